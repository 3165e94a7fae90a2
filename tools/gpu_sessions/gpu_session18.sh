# L2 eviction hints in the superpass: timing per hint mode at n = 30/28, ncu DRAM bytes.
set -x
for m in 0 1 5 9; do timeout 120 python tools/diag_super2.py $m 20 30; done
for m in 0 1 5; do timeout 120 python tools/diag_super2.py $m 20 28; done
for m in 1 5 9; do timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_op_read_hit_rate.pct --clock-control none -k regex:qaa_superpass -s 4 -c 2 python tools/diag_super2.py $m 4 30 2>&1 | grep -E "superpass|duration|dram__|hit_rate"; done
python - <<'PY'
import numpy as np
a0 = np.load("gpurun_out/super_amps_0.npy")
for m in (1, 5):
    a = np.load(f"gpurun_out/super_amps_{m}.npy"); print(m, "max|d|", np.abs(a - a0).max())
PY
