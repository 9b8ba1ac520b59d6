set -u
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "fused_gram" > gpurun_out/g_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/g_tests.log
for v in "" r16; do
  ENKF_LIB_VARIANT=$v timeout 600 python tools/probe/gram_ab.py 0 i8ls,i8fused 5 > gpurun_out/g_ab_$v.json 2> gpurun_out/g_ab_$v.err; echo "ab $v rc=$?"; cat gpurun_out/g_ab_$v.json; tail -2 gpurun_out/g_ab_$v.err
done
ENKF_LIB_VARIANT=gflt timeout 300 python tools/probe/gfl_trace.py 0 > gpurun_out/g_trace.txt 2>&1; head -30 gpurun_out/g_trace.txt
