set -u
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gram_i8_fused -c 1 -f -o gpurun_out/d_fused python tools/probe/gram_ab.py 0 i8fused 1 > gpurun_out/d_ncu.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/d_ncu.log
