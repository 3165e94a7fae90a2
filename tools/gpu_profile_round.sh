# Round artefacts: the bench line, the reference (oracle) line, the launch list of
# the same bench command, one full ncu capture of the fused pass kernels.
set -x
mkdir -p gpurun_out/round
timeout 600 python bench.py > gpurun_out/round/bench.json 2> gpurun_out/round/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/round/bench_reference.json 2> gpurun_out/round/bench_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/round/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/round/ncu_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"qaa_(super)?pass" -s 2 -c 4 -o gpurun_out/round/prof_full python bench.py --steps 1 --warmup 0 --chunk 6 --no-cpu-baseline --no-e2e > gpurun_out/round/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"qaa_pass" -s 2 -c 2 -o gpurun_out/round/prof_twopass python bench.py --steps 1 --warmup 0 --chunk 6 --super 0 --no-cpu-baseline --no-e2e > gpurun_out/round/ncu_twopass.log 2>&1
ls -la gpurun_out/round
