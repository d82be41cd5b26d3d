for v in base hint base hint; do
  if [ $v = base ]; then L=paper_2508_04929_b200/libcgs_b200.so; else L=paper_2508_04929_b200/libcgs_b200_$v.so; fi
  CGS_B200_LIB=$PWD/$L python bench.py --steps 40 --warmup 5 --no-cpu-baseline --sustained-seconds 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', round(d['value']), d['e2e']['value'], {k: round(v,4) for k,v in d['stage_ms'].items()})"
done
