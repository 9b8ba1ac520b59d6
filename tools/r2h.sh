set -u
mkdir -p gpurun_out
ENKF_LIB_VARIANT=gflt timeout 300 python tools/probe/gfl_trace.py 0 > gpurun_out/h_trace_gflt.txt 2>&1; head -8 gpurun_out/h_trace_gflt.txt
ENKF_LIB_VARIANT=nofp timeout 300 python tools/probe/gfl_trace.py 0 > gpurun_out/h_trace_nofp.txt 2>&1; head -8 gpurun_out/h_trace_nofp.txt
ENKF_LIB_VARIANT=nofp timeout 600 python tools/probe/gram_ab.py 0 i8ls,i8fused 3 > gpurun_out/h_ab_nofp.json 2>&1; cat gpurun_out/h_ab_nofp.json | head -c 600
