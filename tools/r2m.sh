set -u
mkdir -p gpurun_out
for n in 64 96 128; do for v in "" lvt lvt0; do echo "variant=$v"; ENKF_LIB_VARIANT=$v python tools/probe/levels_probe.py $n 2>&1 | head -4; done; done > gpurun_out/m_levels.txt 2>&1
cat gpurun_out/m_levels.txt
