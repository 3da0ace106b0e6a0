# quick bench of the cached configs under env variants; prints one table at the end.
# CASES: ';'-separated "label|env|bench args" (default: cfg2/cfg3/cfg4 headline points)
CASES=${CASES:-"cfg2||--efs 70;cfg3||--config cfg3 --efs 100;cfg4||--config cfg4 --efs 4000 --steps 3"}
: > gpurun_out/sweep.txt
IFS=';' read -ra CS <<< "${CASES}"
for c in "${CS[@]}"; do
  IFS='|' read -r label envs args <<< "$c"
  env $envs python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e $args > gpurun_out/sweep_one.json 2> gpurun_out/sweep_one.err
  python -c "import json; d=json.load(open('gpurun_out/sweep_one.json')); print('${label}'.ljust(28), '${envs}'.ljust(36), d['value'], d['roofline']['frac'], d['config']['recall'])" >> gpurun_out/sweep.txt 2>&1 || (echo "${label} FAILED"; tail -3 gpurun_out/sweep_one.err) >> gpurun_out/sweep.txt
done
cat gpurun_out/sweep.txt
