mkdir -p gpurun_out/r2d
make -C paper_2603_06660_b200/csrc variant V=phase FLAGS=-DPAG_PHASE_TIMING > gpurun_out/r2d/make_phase.log 2>&1; echo make=$?
timeout 1200 python -m pytest tests -x -q -m gpu --timeout 400 --timeout-method=thread > gpurun_out/r2d/pytest_gpu.txt 2>&1; echo pytest=$?
tail -15 gpurun_out/r2d/pytest_gpu.txt
for m in fast exact; do timeout 300 python tools/phases.py cfg2 70 $m > gpurun_out/r2d/phase_cfg2_$m.txt 2>&1; echo ph2$m=$?; done
for m in fast exact; do timeout 600 python tools/phases.py cfg3 100 $m > gpurun_out/r2d/phase_cfg3_$m.txt 2>&1; echo ph3$m=$?; done
cat gpurun_out/r2d/phase_*.txt | grep -v "^\[bench\]"
timeout 900 python bench.py --steps 10 --warmup 3 --no-e2e > gpurun_out/r2d/bench_cfg2.json 2> gpurun_out/r2d/bench_cfg2.err; echo cfg2=$?
