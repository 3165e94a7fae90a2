set -x
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
timeout 300 python bench.py --steps 5 --warmup 2 --no-cpu-baseline --no-e2e --kernel 1 > gpurun_out/b4_k1.json 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 30 --csv --log-file gpurun_out/launches4.csv python bench.py --steps 1 --warmup 1 --chunk 10 --no-cpu-baseline --no-e2e > /dev/null 2>&1
