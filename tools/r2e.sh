set -u
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "fused_gram" > gpurun_out/e_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/e_tests.log
for v in "" r16 t3; do
  ENKF_LIB_VARIANT=$v timeout 600 python tools/probe/gram_ab.py 0 i8ls,i8fused 5 > gpurun_out/e_ab_$v.json 2> gpurun_out/e_ab_$v.err; echo "ab $v rc=$?"; cat gpurun_out/e_ab_$v.json; tail -2 gpurun_out/e_ab_$v.err
done
