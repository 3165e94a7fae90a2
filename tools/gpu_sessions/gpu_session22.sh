# fewer group barriers (leading WAR barrier, warp-local PB->PC in group 0): parity + timing
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "super or tma or pass or n30" 2>&1 | tail -3
for m in 1 0; do timeout 120 python tools/diag_super2.py $m 20 30; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:qaa_superpass -s 4 -c 1 -o gpurun_out/super5_full python tools/diag_super2.py 1 4 > gpurun_out/super5_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:qaa_pass_tma -s 6 -c 2 -o gpurun_out/pass5_full python tools/diag_super2.py 0 4 > gpurun_out/pass5_ncu.log 2>&1
tail -1 gpurun_out/super5_ncu.log gpurun_out/pass5_ncu.log
