for r in 1 2; do for e in "$@"; do
  env $e python bench.py --steps 60 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$e', round(d['value']), 'e2e', round(d['e2e']['value']), {k: round(v,4) for k,v in d['stage_ms'].items()})"
done; done
