set -u
mkdir -p gpurun_out
for n in 64 96 128; do python tools/probe/levels_probe.py $n; ENKF_LIB_VARIANT=lvt python tools/probe/levels_probe.py $n; done > gpurun_out/j_levels.txt 2>&1
cat gpurun_out/j_levels.txt
