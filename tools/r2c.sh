set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "int8_gram or fused_gram or level_split" > gpurun_out/c_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/c_tests.log
timeout 600 python tools/probe/gram_ab.py 0 i8ls,i8fused 5 > gpurun_out/c_gram_ab.json 2> gpurun_out/c_gram_ab.err; echo "ab rc=$?"; cat gpurun_out/c_gram_ab.json; tail -3 gpurun_out/c_gram_ab.err
