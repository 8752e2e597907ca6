"""Build debug variants: libhm_timing.so (phase timestamps) and libhm_stopK.so (k_bucket cut after mark K)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from concurrent.futures import ThreadPoolExecutor
from paper_2508_11443_b200 import _build
jobs = [("timing", ["HM_PHASE_TIMING"])] + [(f"stop{k}", [f"HM_STOP_AFTER={k}"]) for k in range(1, 8)]
jobs += [(a, b.split(",")) for a, b in (x.split("=", 1) for x in sys.argv[1:])]
with ThreadPoolExecutor(8) as ex:
    for r in ex.map(lambda j: _build.build_variant(*j), jobs):
        print(r)
