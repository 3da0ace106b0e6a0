mkdir -p gpurun_out/r2i
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/r2i/pytest_gpu.txt 2>&1; echo pytest=$?; tail -2 gpurun_out/r2i/pytest_gpu.txt
NEW=paper_2603_06660_b200/libpag_gpu.so; OLD=build/lib_base.so
for c in "cfg2 70 exact" "cfg2 70 warp-tree"; do timeout 900 python tools/ab_time.py $c $OLD $NEW 3; done | tee gpurun_out/r2i/ab.jsonl
timeout 900 python tools/ab_cons.py $OLD $NEW 3 | tee -a gpurun_out/r2i/ab.jsonl
