# cfg-4 (2M x 512, K = 1000): bench line, then the concurrency experiment:
# resident blocks per SM capped at 6/4/3/2 -> time and DRAM bytes per launch
mkdir -p gpurun_out/r2e
timeout 1800 python bench.py --config cfg4 --steps 5 --warmup 3 > gpurun_out/r2e/bench_cfg4.json 2> gpurun_out/r2e/bench_cfg4.err; echo cfg4=$?
tail -3 gpurun_out/r2e/bench_cfg4.err
for b in 6 4 3 2; do
  PAG_GPU_MAX_BPS=$b timeout 600 python bench.py --config cfg4 --efs 4000 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2e/occ_$b.json 2> gpurun_out/r2e/occ_$b.err; echo occ$b=$?
  PAG_GPU_MAX_BPS=$b timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:pag_search -s 3 -c 1 --csv python bench.py --config cfg4 --efs 4000 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2e/ncu_occ_$b.csv 2> gpurun_out/r2e/ncu_occ_$b.err; echo ncu$b=$?
done
for b in 6 4 3 2; do python -c "
import json; d=json.load(open('gpurun_out/r2e/occ_$b.json')); print($b, d['value'], d['ms_per_step'], d['roofline']['frac'])"; grep -E "dram__bytes|gpu__time|lts__t" gpurun_out/r2e/ncu_occ_$b.csv | cut -d, -f12- ; done
