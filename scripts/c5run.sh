OUT=gpurun_out/${TAG:-c5}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
libs=""
for v in $VARIANTS; do
  tag=${v%%:*}; defs=${v#*:}
  python -c "
import sys; sys.path.insert(0,'.')
from paper_2508_11443_b200 import _build
print(_build.build_variant('$tag', '$defs'.split(',')))" >> $OUT/build.log 2>&1
  libs="$libs paper_2508_11443_b200/libhm_$tag.so"
done
python scripts/c5_variants.py $libs 2>&1 | tee $OUT/c5.txt
