ncu --set full --import-source on --clock-control none -k regex:"wbound_chunk|prepare_kernel" -s 4 -c 2 -o gpurun_out/wb python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
CGS_GRAPHS=0 ncu --set full --import-source on --clock-control none -k regex:"epilogue_adam" -s 2 -c 1 -o gpurun_out/epi python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
