# Superpass v2 (seg fix) parity + timing; L2 promotion experiment on the default plan.
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "super" 2>&1 | tail -4
for m in 0 1 3; do timeout 120 python tools/diag_super2.py $m 20; done
for pr in 64 128 256; do QAA_L2_PROMO=$pr timeout 120 python tools/diag_super2.py 0 20; QAA_L2_PROMO=$pr timeout 120 python tools/diag_super2.py 1 20; done
python - <<'PY'
import numpy as np
a0 = np.load("gpurun_out/super_amps_0.npy")
for m in (1, 3):
    a = np.load(f"gpurun_out/super_amps_{m}.npy"); print(m, "max|d|", np.abs(a - a0).max())
PY
timeout 600 ncu --set full --clock-control none --import-source on -k regex:qaa_superpass -s 4 -c 2 -o gpurun_out/super3_full python tools/diag_super2.py 1 4 > gpurun_out/super3_ncu.log 2>&1
tail -2 gpurun_out/super3_ncu.log
