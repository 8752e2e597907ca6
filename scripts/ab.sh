#!/bin/bash
# A/B pass on the GPU box: parity tests of the default build, per-kernel times
# of the default and the variant builds (VARIANTS="tag:DEFINE[,DEFINE] ..."),
# quick 2^26 / 2^24-bytes timings; an ncu capture of k_bucket when NCU=1.
OUT=gpurun_out/${TAG:-ab}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -20 $OUT/build.log; exit 1; }
libs=""
for v in $VARIANTS; do
  tag=${v%%:*}; defs=${v#*:}
  python -c "
import sys; sys.path.insert(0,'.')
from paper_2508_11443_b200 import _build
print(_build.build_variant('$tag', '$defs'.split(',')))" >> $OUT/build.log 2>&1
  libs="$libs paper_2508_11443_b200/libhm_$tag.so"
done
[ -z "$NOTEST" ] && { timeout 900 python -m pytest tests/${TESTS:-test_gpu_parity.py} -x -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log; tail -3 $OUT/pytest.log; }
timeout 600 python scripts/variant_times.py $libs 2>&1 | tee $OUT/variants.txt
timeout 300 python scripts/quick_bench.py 26 2>&1 | tee $OUT/quick26.txt
[ -n "$BYTES" ] && timeout 600 python scripts/bytes_build_variants.py $libs 2>&1 | tee $OUT/bytes_variants.txt
if [ -n "$NCU" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_bucket" -c 1 -o $OUT/kb python scripts/prof_once.py 26 > $OUT/ncu.log 2>&1
fi
true
if [ -n "$TIMING" ]; then
  python -c "
import sys; sys.path.insert(0,'.')
from paper_2508_11443_b200 import _build
_build.build_variant('timing', ['HM_PHASE_TIMING'] + [d for d in '${TIMING_DEFS}'.split(',') if d])" >> $OUT/build.log 2>&1
  timeout 300 python scripts/phase_times.py 26 2>&1 | tee $OUT/phases.txt
fi
[ -n "$LBYTES" ] && timeout 600 python scripts/lookup_bytes_variants.py $libs 2>&1 | tee $OUT/lookup_bytes_variants.txt
true
