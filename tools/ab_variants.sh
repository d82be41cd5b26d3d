for v in base; do
  if [ $v = base ]; then L=paper_2508_04929_b200/libcgs_b200.so; else L=paper_2508_04929_b200/libcgs_b200_$v.so; fi
  CGS_B200_LIB=$PWD/$L python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', round(d['value']), d['stage_ms'])"
done
