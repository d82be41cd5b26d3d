timeout 600 python -m pytest tests -m gpu -x -q -k "peer or nccl" 2>&1 | tail -30
