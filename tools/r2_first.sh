set -u
mkdir -p gpurun_out
nproc > gpurun_out/r2a_box.txt; free -g >> gpurun_out/r2a_box.txt; nvidia-smi -L >> gpurun_out/r2a_box.txt; lscpu | head -20 >> gpurun_out/r2a_box.txt
ls /usr/include/nccl* /usr/local/cuda/include/nccl* 2>&1 >> gpurun_out/r2a_box.txt
python -m pytest tests -m gpu -q -x > gpurun_out/r2a_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2a_tests.log
python bench.py > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err; echo "bench rc=$?"; cat gpurun_out/r2a_bench.json | head -c 600
