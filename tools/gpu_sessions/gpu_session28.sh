# functional multi-rank runs on one GPU (ranks share cuda:0): bench N=2 and the reference arm
set -x
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --share-gpu --steps 2 --warmup 1 --chunk 10 --no-cpu-baseline > gpurun_out/b_n2.json 2> gpurun_out/b_n2.err; echo rc=$?; cat gpurun_out/b_n2.json | cut -c1-400; tail -5 gpurun_out/b_n2.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > gpurun_out/b_ref_n2.json 2> gpurun_out/b_ref_n2.err; echo rc=$?; cat gpurun_out/b_ref_n2.json | cut -c1-300
