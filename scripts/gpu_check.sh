#!/bin/bash
# One GPU pass: build, gpu tests, smoke, bench, ncu launch list + full capture of the hot kernels.
set -x
OUT=gpurun_out/${TAG:-run}
mkdir -p $OUT
nvidia-smi -L > $OUT/gpu.txt
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
[ -z "$NOTEST" ] && { timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log; }
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 600 python bench.py --impl reference > $OUT/bench_ref.json 2> $OUT/bench_ref.err
if [ -n "$NCU" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 1 --no-configs --no-e2e --no-cpu-baseline > $OUT/bench_ncu.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_lookup_u64|k_bucket|k_split" -c 7 -o $OUT/full python scripts/prof_once.py 26 > $OUT/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_lookup_bytes|k_bucket|k_split|k_fingerprint" -c 8 -o $OUT/full_bytes python scripts/prof_once.py 24 bytes > $OUT/ncu_full_bytes.log 2>&1
fi
timeout 600 python scripts/bench_configs.py > $OUT/configs.jsonl 2> $OUT/configs.err
timeout 300 python scripts/rounds_bench.py > $OUT/rounds_ablation.jsonl 2> $OUT/rounds.err
tail -3 $OUT/pytest_gpu.log; tail -2 $OUT/smoke.log; cat $OUT/bench.json $OUT/bench_ref.json
