#!/bin/bash
# One GPU session's evidence: GPU tests, the default bench line, the ncu launch
# list of the same bench command, and ncu --set full captures of the Gram kernels.
# Outputs in gpurun_out/ (copy the summaries to profiles/).
set -u
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/cap_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/cap_tests.log
python -m pytest tests/test_fullsize_gpu.py -m gpu -q -s 2>&1 | grep -a "full-size parity" > gpurun_out/cap_fullsize.txt
python bench.py > gpurun_out/cap_bench.json 2> gpurun_out/cap_bench.err; echo "bench rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cap_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/cap_ncu_bench.log 2>&1; echo "ncu list rc=$?"
ncu --set full --import-source on --clock-control none -k regex:"gram_i8_(mma|slice)" -c 2 -f -o gpurun_out/cap_gram_full \
    python tools/probe/g8_time.py 23 26 > gpurun_out/cap_gram_full.log 2>&1; echo "ncu full rc=$?"
