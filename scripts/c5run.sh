OUT=gpurun_out/c5; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
python -c "
import sys; sys.path.insert(0,'.')
from paper_2508_11443_b200 import _build
print(_build.build_variant('plainmul', ['HM_PLAIN_MUL']))" >> $OUT/build.log 2>&1
python scripts/c5_variants.py paper_2508_11443_b200/libhm_plainmul.so paper_2508_11443_b200/libhm_r01.so 2>&1 | tee $OUT/c5.txt
