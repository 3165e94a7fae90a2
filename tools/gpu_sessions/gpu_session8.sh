set -x
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "strang or sweep" 2>&1 | tail -8
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 200 python bench.py --steps 5 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/b8.json 2>&1
