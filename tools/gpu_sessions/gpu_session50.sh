set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "super or bitwise or n30" 2>&1 | tail -2
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/b50.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/b50.json')); print(d['value'], d['e2e']['value'], d['clocks']['sm_mhz'], d['roofline']['launches'], d['roofline']['all_pass_launches'], round(d['roofline']['frac'],3))"
