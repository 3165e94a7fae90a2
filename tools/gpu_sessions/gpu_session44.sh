set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_sharded.py -m gpu -x -q -k "energy or n30 or max_size or sharded or sweep" 2>&1 | tail -3
timeout 600 python tools/bench_energy.py
