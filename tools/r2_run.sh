# round-2 GPU session: tests, bench (config 5 + configs 1-3)
set -u
mkdir -p gpurun_out
T=${1:-b}
python -m pytest tests -m gpu -q -x -s -p no:randomly > gpurun_out/${T}_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/${T}_tests.log
grep -a "full-size parity" gpurun_out/${T}_tests.log > gpurun_out/${T}_fullsize.txt
python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc=$?"; tail -2 gpurun_out/${T}_bench.err
for c in 1 2 3; do python bench.py --config $c --steps 200 --warmup 20 --e2e-steps 20 > gpurun_out/${T}_bench_c$c.json 2>> gpurun_out/${T}_bench.err; echo "c$c rc=$?"; done
