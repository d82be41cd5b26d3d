nproc
timeout 900 python -m pytest tests -m gpu -x -q -k "full_c2_batch" --durations=3 2>&1 | tail -8
