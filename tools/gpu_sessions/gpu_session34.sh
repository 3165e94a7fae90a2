timeout 900 python bench.py > gpurun_out/b34.json 2> gpurun_out/b34.err; cat gpurun_out/b34.json; tail -2 gpurun_out/b34.err
