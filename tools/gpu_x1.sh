# chain-interleaved reference-order distances: parity suite, then A/B against the previous build
D=gpurun_out/x1; mkdir -p $D
timeout 1500 python -m pytest tests -x -q -m gpu > $D/pytest_gpu.txt 2>&1; echo pytest=$?; tail -3 $D/pytest_gpu.txt
NEW=paper_2603_06660_b200/libpag_gpu.so; OLD=build/lib_base.so
for c in "cfg2 70 exact" "cfg2 70 warp-tree" "cfg1 30 exact"; do timeout 1200 python tools/ab_time.py $c $OLD $NEW 3; done | tee $D/ab.jsonl
timeout 900 python tools/ab_cons.py $OLD $NEW 3 | tee -a $D/ab.jsonl
