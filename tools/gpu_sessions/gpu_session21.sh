# full ncu of the default superpass (n = 30) with source-level stall info
set -x
timeout 600 ncu --set full --clock-control none --import-source on -k regex:qaa_superpass -s 4 -c 1 -o gpurun_out/super4_full python tools/diag_super2.py 1 4 > gpurun_out/super4_ncu.log 2>&1
tail -2 gpurun_out/super4_ncu.log
