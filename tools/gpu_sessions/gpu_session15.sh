# Superpass diagnosis: timing per mode + sampled amplitude agreement + one ncu capture.
set -x
for m in 0 1 3 5 7; do timeout 120 python tools/diag_super2.py $m 20; echo "rc=$?"; done
python - <<'PY'
import numpy as np
a0 = np.load("gpurun_out/super_amps_0.npy")
for m in (1, 3, 5, 7):
    try:
        a = np.load(f"gpurun_out/super_amps_{m}.npy"); print(m, "max|d|", np.abs(a - a0).max())
    except Exception as e: print(m, e)
PY
timeout 600 ncu --set full --clock-control none --import-source on -k regex:qaa_superpass -s 4 -c 2 -o gpurun_out/super_full python tools/diag_super2.py 1 4 > gpurun_out/super_ncu.log 2>&1
tail -3 gpurun_out/super_ncu.log
