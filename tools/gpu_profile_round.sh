# Round artefacts (run under gpurun on one B200): the bench line, the reference
# (oracle) line, the launch list of the bench command, one full ncu capture of
# the L2-blocked step, of the two-pass plan's kernels, and of the small-state
# single-launch engines (warp-tile n = 16, cluster-resident n = 14).
#   bash tools/gpu_profile_round.sh r02
set -x
R=${1:-r02}
O=gpurun_out/$R
mkdir -p $O
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"qaa_superpass" -s 2 -c 2 -o $O/prof_super python bench.py --steps 1 --warmup 0 --chunk 6 --no-cpu-baseline --no-e2e > $O/ncu_super.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"qaa_pass" -s 2 -c 2 -o $O/prof_twopass python bench.py --steps 1 --warmup 0 --chunk 6 --super 0 --no-cpu-baseline --no-e2e > $O/ncu_twopass.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"qaa_quad_evolve|qaa_warp_evolve|qaa_cluster_evolve" -c 3 -o $O/prof_small python tools/profile_small.py > $O/ncu_small.log 2>&1
timeout 900 python tools/bench_configs.py > $O/configs.jsonl 2> $O/configs.err
ls -la $O
