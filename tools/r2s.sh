set -u
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "int8_gram or fused_gram" > gpurun_out/s_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/s_tests.log
ENKF_LIB_VARIANT=gflt timeout 300 python tools/probe/gfl_trace.py 0 > gpurun_out/s_trace.txt 2>&1; sed -n 2,8p gpurun_out/s_trace.txt
timeout 600 python tools/probe/gram_ab.py 0 i8ls,i8fused 4 > gpurun_out/s_ab.json 2>&1; python -c "import json; d=json.load(open('gpurun_out/s_ab.json')); print({m: (round(d[m]['gram_ms_med'],2), round(d[m]['step_ms_med'],2), d[m]['gram_ms']) for m in ('i8ls','i8fused')}, d.get('gram_i8fused_vs_i8ls'))"
