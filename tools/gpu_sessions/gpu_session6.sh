set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -3
for g in 0 1 2; do
timeout 300 python bench.py --steps 5 --warmup 2 --no-cpu-baseline --no-e2e --tma-groups $g > gpurun_out/b6_g${g}.json 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 20 --csv --log-file gpurun_out/launches6_g${g}.csv python bench.py --steps 1 --warmup 1 --chunk 10 --no-cpu-baseline --no-e2e --tma-groups $g > /dev/null 2>&1
done
