set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "super or tma or pass or n30 or bitwise or strang or driver" 2>&1 | tail -3
for m in 1 1 1; do timeout 120 python tools/diag_super2.py $m 20 30; done
timeout 120 python tools/diag_super2.py 0 20 30
timeout 120 python tools/diag_super2.py 1 50 24
