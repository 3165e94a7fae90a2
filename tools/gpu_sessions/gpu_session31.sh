set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "super" 2>&1 | tail -2
timeout 600 python tools/bench_configs.py 2>/dev/null | cut -c1-200
