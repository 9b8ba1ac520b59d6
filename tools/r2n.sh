set -u
mkdir -p gpurun_out
for rep in 1 2; do for v in "" c32; do
  ENKF_LIB_VARIANT=$v python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-extras > gpurun_out/n_b_${v}_$rep.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/n_b_${v}_$rep.json')); print('$v', $rep, round(d['value'],2), {k: round(v,2) for k,v in d['kernels_ms'].items()}, round(d['energy_j_per_step'],1), d['clocks']['sm_mhz'])"
done; done
ENKF_LIB_VARIANT=c32 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "anomaly or tensor_core or config_goldens or analysis_vs_oracle" 2>&1 | tail -2
