#!/bin/bash
# Full GPU pass: build, every gpu test, smoke, bench (ours + reference), the
# --gpus 2 launcher check on a 1-GPU box, host facts.
OUT=gpurun_out/${TAG:-pass}
mkdir -p $OUT
{ nvidia-smi -L; nproc; free -g | head -2; } > $OUT/host.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
[ -z "$NOTEST" ] && { timeout 1500 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log; tail -4 $OUT/pytest_gpu.log; }
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"; cat $OUT/bench.json | cut -c1-3000
[ -n "$REF" ] && { timeout 600 python bench.py --impl reference > $OUT/bench_ref.json 2> $OUT/bench_ref.err; cut -c1-400 $OUT/bench_ref.json; }
timeout 120 python bench.py --gpus 2 > $OUT/bench_g2.out 2> $OUT/bench_g2.err; echo "bench --gpus 2 rc=$?"; cat $OUT/bench_g2.err | tail -2
true
