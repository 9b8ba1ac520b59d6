#!/bin/bash
# One GPU session's evidence (round 2): GPU tests, the default bench line, the ncu
# launch list of the same bench command, and ncu --set full captures of the Gram
# passes (config 5) and of the anomaly kernel (config-4 rows).  Outputs in
# gpurun_out/${TAG}_* (copy the summaries to profiles/).
set -u
T=${1:-cap}
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -s > gpurun_out/${T}_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/${T}_tests.log
grep -a "full-size parity" gpurun_out/${T}_tests.log > gpurun_out/${T}_fullsize.txt
python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-extras > gpurun_out/${T}_ncu_bench.log 2>&1; echo "ncu list rc=$?"
ncu --set full --import-source on --clock-control none -k regex:"gram_i8_(mma_ls|slice)" -c 2 -f -o gpurun_out/${T}_gram_full \
    python tools/probe/g8_time.py 23 26 > gpurun_out/${T}_gram_full.log 2>&1; echo "ncu gram rc=$?"
ncu --set full --import-source on --clock-control none -k regex:"anomaly_i8" -c 1 -f -o gpurun_out/${T}_anom_full \
    python tools/probe/i8_only.py 24 1 > gpurun_out/${T}_anom_full.log 2>&1; echo "ncu anomaly rc=$?"
