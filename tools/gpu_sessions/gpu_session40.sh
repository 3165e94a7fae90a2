set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "super or bitwise" 2>&1 | tail -2
for m in 1 1; do timeout 120 python tools/diag_super2.py $m 20 30; done
timeout 120 python tools/diag_super2.py 1 50 28
