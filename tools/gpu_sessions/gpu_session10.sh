set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
for sp in 2 1; do
timeout 200 python bench.py --steps 5 --warmup 2 --no-cpu-baseline --no-e2e --step-spanning $sp > gpurun_out/b10_sp${sp}.json 2>&1
done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 16 --csv --log-file gpurun_out/launches10.csv python bench.py --steps 1 --warmup 1 --chunk 6 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 300 python tools/bench_configs.py > gpurun_out/configs.jsonl 2>&1
