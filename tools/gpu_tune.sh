# compare PAG_GPU_TUNE variants on the cached cfg2 index (efS fixed)
for t in ${TUNES:-0 1 2 3}; do
  for rep in 1 2; do
    PAG_GPU_TUNE=$t python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --efs ${EFS:-70} ${EXTRA:-} 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('tune', $t, 'rep', $rep, d['value'], d['roofline']['frac'])"
  done
done
