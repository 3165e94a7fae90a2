set -x
timeout 1200 python -m pytest tests/test_sharded.py -m gpu -x -q 2>&1 | tail -5
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --share-gpu --steps 2 --warmup 1 --chunk 10 --no-cpu-baseline --no-e2e > gpurun_out/b_n2.json 2> gpurun_out/b_n2.err; echo rc=$?; python -c "
import json; d=json.load(open('gpurun_out/b_n2.json')); print(d['value'], d['roofline']['kernel'], d['roofline']['launches'], d['roofline']['avg_launch_ms'])"; tail -3 gpurun_out/b_n2.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --share-gpu --steps 2 --warmup 1 --chunk 10 --no-cpu-baseline --no-e2e --super 0 > gpurun_out/b_n2s0.json 2> gpurun_out/b_n2s0.err; python -c "
import json; d=json.load(open('gpurun_out/b_n2s0.json')); print('super0', d['value'])"
