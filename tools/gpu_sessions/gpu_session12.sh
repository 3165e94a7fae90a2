set -x
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "driver" 2>&1 | tail -4
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
