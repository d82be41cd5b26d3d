# A/B of environment switches on the C2 bench: bash tools/ab_env.sh "VAR=1" "VAR=0" ...
for e in "$@"; do
  env $e python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$e', round(d['value']), 'e2e', round(d['e2e']['value']), d['stage_ms'])"
done
