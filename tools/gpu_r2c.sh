# phase accounting (cfg2 both modes, cfg3), cfg3 bench, cfg2 parity examples
mkdir -p gpurun_out/r2c
make -C paper_2603_06660_b200/csrc variant V=phase FLAGS=-DPAG_PHASE_TIMING > gpurun_out/r2c/make_phase.log 2>&1; echo make=$?
timeout 900 python bench.py --config cfg3 --steps 10 --warmup 3 > gpurun_out/r2c/bench_cfg3.json 2> gpurun_out/r2c/bench_cfg3.err; echo cfg3=$?
for m in fast exact; do timeout 300 python tools/phases.py cfg2 70 $m > gpurun_out/r2c/phase_cfg2_$m.txt 2>&1; echo ph2$m=$?; done
for m in fast exact; do timeout 300 python tools/phases.py cfg3 100 $m > gpurun_out/r2c/phase_cfg3_$m.txt 2>&1; echo ph3$m=$?; done
cat gpurun_out/r2c/phase_*.txt
timeout 900 python bench.py --steps 10 --warmup 3 --no-e2e > gpurun_out/r2c/bench_cfg2.json 2> gpurun_out/r2c/bench_cfg2.err; echo cfg2=$?
