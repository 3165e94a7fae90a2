# superpass default hints: parity + bench comparison
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "super" 2>&1 | tail -3
timeout 300 python bench.py --no-cpu-baseline --no-e2e --super 0 > gpurun_out/b_s0.json 2>&1; cat gpurun_out/b_s0.json | cut -c1-200
timeout 300 python bench.py --no-cpu-baseline --no-e2e --super 1 > gpurun_out/b_s1.json 2>&1; cat gpurun_out/b_s1.json | cut -c1-200
timeout 300 python bench.py --no-cpu-baseline --no-e2e --super 1 --chunk 100 --steps 4 > gpurun_out/b_s1c100.json 2>&1; cat gpurun_out/b_s1c100.json | cut -c1-200
