set -u
mkdir -p gpurun_out
for n in 2 3 7 20 31 64 96 97 128; do for m in single cluster; do echo -n "$m "; ENKF_LEVELS=$m python tools/probe/levels_probe.py $n 2>&1 | head -1; done; done > gpurun_out/o_levels.txt 2>&1
cat gpurun_out/o_levels.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "levels or singular or config or random_systems" > gpurun_out/o_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/o_tests.log
for c in 2 3; do python bench.py --config $c --steps 200 --warmup 20 --e2e-steps 20 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($c, round(d['value']), {k: round(v*1e3,1) for k,v in d['kernels_ms'].items()})"; done
