# final check of the committed tree: the driver's sequence, then the reference-order lines of cfg-3 / cfg-4
bash tools/gpu_driver_mirror.sh
R=gpurun_out/mirror
timeout 1500 python bench.py --config cfg3 --dist exact --steps 10 --warmup 3 --no-cpu-baseline > $R/bench_cfg3_exact.json 2> $R/bench_cfg3_exact.err; echo cfg3x=$?
timeout 2400 python bench.py --config cfg4 --dist exact --steps 5 --warmup 3 --no-cpu-baseline > $R/bench_cfg4_exact.json 2> $R/bench_cfg4_exact.err; echo cfg4x=$?
for c in cfg3 cfg4; do python -c "
import json; d=json.load(open('$R/bench_${c}_exact.json')); print('$c exact', d['value'], d['roofline']['frac'], d['roofline']['traffic'], d['e2e']['value'])"; done
