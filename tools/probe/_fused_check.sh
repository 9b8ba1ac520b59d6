timeout 300 python tools/probe/g8_ab.py 23 26 3 2>&1 | tail -1
timeout 300 python tools/probe/g8_ab.py 21 24 3 2>&1 | tail -1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_sharded_gpu.py -q -x 2>&1 | tail -2
ncu --set full --import-source on --clock-control none -k regex:gram_i8_fused -c 1 -f -o gpurun_out/fused_full2 python tools/probe/g8_time.py 21 24 > gpurun_out/fused_full2.log 2>&1; echo ncu rc=$?
