python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo rc=$?; tail -2 gpurun_out/bench.err
