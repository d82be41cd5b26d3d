# One profiling round on a B200 (gpurun): bench, reference arm, sweep, C3 epoch, launch list,
# full ncu captures of one step's kernels, GPU tests with the parity-margin log.  Outputs under
# gpurun_out/ (copy the summaries to profiles/).
set -x
python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
python tools/sweep.py --out gpurun_out/sweep.json > gpurun_out/sweep.log 2>&1
python tools/epoch_c3.py --out gpurun_out/epoch_c3.json > gpurun_out/epoch_c3.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --sustained-seconds 0 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:"wbound_chunk|raster_fwd_atomic|ctf_mse_spec|raster_bwd_region|epilogue_adam" -s 20 -c 5 -o gpurun_out/prof_full python bench.py --steps 1 --warmup 4 --no-cpu-baseline --sustained-seconds 0 > gpurun_out/ncu_full.log 2>&1
CGS_MARGIN_LOG=$PWD/gpurun_out/parity_margins.tsv python -m pytest tests -m gpu -q > gpurun_out/gputest.log 2>&1
tail -c 400 gpurun_out/bench_full.json
