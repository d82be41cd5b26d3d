CGS_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 5 --warmup 3 --sustained-seconds 0.5 > gpurun_out/bench2.json 2> gpurun_out/bench2.err; echo rc=$?
tail -5 gpurun_out/bench2.err
cat gpurun_out/bench2.json | tail -c 600
CGS_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 2 --steps 5 --warmup 3 --scaling strong --sustained-seconds 0 > gpurun_out/bench2s.json 2> gpurun_out/bench2s.err; echo rc=$?
tail -c 300 gpurun_out/bench2s.json
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29613 bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > gpurun_out/bench2r.json 2> gpurun_out/bench2r.err; echo rc=$?
tail -c 300 gpurun_out/bench2r.json
