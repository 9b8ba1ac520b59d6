set -u
mkdir -p gpurun_out
for n in 64 96 128; do for v in "" ldl1 lvt lvt1; do echo "variant=$v"; ENKF_LIB_VARIANT=$v python tools/probe/levels_probe.py $n | head -3; done; done > gpurun_out/l_levels.txt 2>&1
cat gpurun_out/l_levels.txt | grep -v "^[0-9]* gather" 
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_host_logic.py tests/test_localized.py tests/test_lorenz96.py -q -x > gpurun_out/l_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/l_tests.log
