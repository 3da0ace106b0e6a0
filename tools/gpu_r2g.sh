mkdir -p gpurun_out/r2g
timeout 1200 python -m pytest tests -x -q -m gpu --timeout 400 --timeout-method=thread > gpurun_out/r2g/pytest_gpu.txt 2>&1; echo pytest=$?
tail -2 gpurun_out/r2g/pytest_gpu.txt
NEW=paper_2603_06660_b200/libpag_gpu.so; OLD=build/lib_base.so
for c in "cfg2 70 warp-tree" "cfg2 70 exact"; do timeout 900 python tools/ab_time.py $c $OLD $NEW 3; done | tee gpurun_out/r2g/ab.jsonl
timeout 1200 python bench.py --config cfg3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
for c in "cfg3 100 warp-tree" "cfg3 100 exact"; do timeout 900 python tools/ab_time.py $c $OLD $NEW 3; done | tee -a gpurun_out/r2g/ab.jsonl
