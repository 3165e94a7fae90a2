# Superpass v2: parity, timing per mode, ncu capture; stride/TLB microbenchmark.
set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "super" 2>&1 | tail -4
for m in 0 1 3; do timeout 120 python tools/diag_super2.py $m 20; echo "rc=$?"; done
python - <<'PY'
import numpy as np
a0 = np.load("gpurun_out/super_amps_0.npy")
for m in (1, 3):
    try:
        a = np.load(f"gpurun_out/super_amps_{m}.npy"); print(m, "max|d|", np.abs(a - a0).max())
    except Exception as e: print(m, e)
PY
timeout 600 ncu --set full --clock-control none --import-source on -k regex:qaa_superpass -s 4 -c 2 -o gpurun_out/super2_full python tools/diag_super2.py 1 4 > gpurun_out/super2_ncu.log 2>&1
tail -2 gpurun_out/super2_ncu.log
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/mb tools/microbench/mb.cu && timeout 300 /tmp/mb 2>&1 | grep -v "^DFMA\|^SHFL"
