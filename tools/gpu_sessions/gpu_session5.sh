set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -6
timeout 300 python bench.py --steps 5 --warmup 2 --no-cpu-baseline --no-e2e --kernel 1 > gpurun_out/b5_k1.json 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 30 --csv --log-file gpurun_out/launches5.csv python bench.py --steps 1 --warmup 1 --chunk 10 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:qaa_pass_tma -s 4 -c 4 -o gpurun_out/prof_tma5 python bench.py --steps 1 --warmup 0 --chunk 6 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full5.log 2>&1
