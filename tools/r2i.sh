set -u
mkdir -p gpurun_out
for v in r16t sc12 sc12n; do
ENKF_LIB_VARIANT=$v timeout 300 python tools/probe/gfl_trace.py 0 > gpurun_out/i_trace_$v.txt 2>&1; echo $v; head -8 gpurun_out/i_trace_$v.txt | tail -6
ENKF_LIB_VARIANT=$v timeout 600 python tools/probe/gram_ab.py 0 i8ls,i8fused 3 > gpurun_out/i_ab_$v.json 2>&1; python -c "import json; d=json.load(open('gpurun_out/i_ab_$v.json')); print({m: (d[m]['gram_ms_med'], d[m]['step_ms_med']) for m in ('i8ls','i8fused')})"
done
