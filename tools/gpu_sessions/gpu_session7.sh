set -x
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "super" 2>&1 | tail -8
timeout 150 python bench.py --steps 5 --warmup 2 --no-cpu-baseline --no-e2e --super 1 > gpurun_out/b7_s1.json 2>&1
timeout 150 python bench.py --steps 5 --warmup 2 --no-cpu-baseline --no-e2e --super 5 > gpurun_out/b7_s5.json 2>&1
timeout 150 python bench.py --steps 5 --warmup 2 --no-cpu-baseline --no-e2e --super 3 > gpurun_out/b7_s3.json 2>&1
timeout 200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -c 16 --csv --log-file gpurun_out/launches7.csv python bench.py --steps 1 --warmup 1 --chunk 6 --no-cpu-baseline --no-e2e > /dev/null 2>&1
