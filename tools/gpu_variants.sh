# run the cached cfg2 bench (fixed efS) under several env settings; VARIANTS separated by ';'
IFS=';' read -ra VS <<< "${VARIANTS}"
for v in "${VS[@]}"; do
  env $v python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --efs ${EFS:-70} ${EXTRA:-} 2>gpurun_out/var.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v'.ljust(60), d['value'], d['roofline']['frac'], d['config']['recall'])" || tail -3 gpurun_out/var.err
done
