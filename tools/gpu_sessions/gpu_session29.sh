set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "bitwise" 2>&1 | tail -3
