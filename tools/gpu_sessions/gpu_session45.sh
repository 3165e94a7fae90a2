set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "max_size or bitwise or super" 2>&1 | tail -3
for m in 1 0; do timeout 300 python tools/diag_super2.py $m 10 31; done
for m in 1 0; do timeout 300 python tools/diag_super2.py $m 6 32; done
