"""Build tuning variants of libstragglar.so into build/variants/ (travels with gpurun)."""
import os
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2505_23523_b200 import build as B  # noqa: E402

VARIANTS_ALL = {
    "s3_16k": ["STRAGGLAR_STAGES=3", "STRAGGLAR_STAGE_BYTES=16384"],
    "s4_12k": ["STRAGGLAR_STAGES=4", "STRAGGLAR_STAGE_BYTES=12288"],
    "s6_8k": ["STRAGGLAR_STAGES=6", "STRAGGLAR_STAGE_BYTES=8192"],
    "s2_24k": ["STRAGGLAR_STAGES=2", "STRAGGLAR_STAGE_BYTES=24576"],
    "s4_16k": ["STRAGGLAR_STAGES=4", "STRAGGLAR_STAGE_BYTES=16384"],
    "s3_32k": ["STRAGGLAR_STAGES=3", "STRAGGLAR_STAGE_BYTES=32768"],
    "s3_16k_t512": ["STRAGGLAR_STAGES=3", "STRAGGLAR_STAGE_BYTES=16384", "STRAGGLAR_THREADS=512", "STRAGGLAR_MIN_BLOCKS=2"],
    "s3_8k_t128": ["STRAGGLAR_STAGES=3", "STRAGGLAR_STAGE_BYTES=8192", "STRAGGLAR_THREADS=128", "STRAGGLAR_MIN_BLOCKS=8"],
}
VARIANTS_LAG = {
    "lag0_s3": ["STRAGGLAR_TMA_LAG=0"],
    "lag1_s3": ["STRAGGLAR_TMA_LAG=1"],
    "lag1_s4_12k": ["STRAGGLAR_TMA_LAG=1", "STRAGGLAR_STAGES=4", "STRAGGLAR_STAGE_BYTES=12288"],
    "lag1_s4_16k": ["STRAGGLAR_TMA_LAG=1", "STRAGGLAR_STAGES=4", "STRAGGLAR_STAGE_BYTES=16384"],
    "lag1_s6_8k": ["STRAGGLAR_TMA_LAG=1", "STRAGGLAR_STAGES=6", "STRAGGLAR_STAGE_BYTES=8192"],
}
VARIANTS_LL = {
    "ll_gentle32": ["STRAGGLAR_LL_GENTLE=32"],
    "ll_gentle200": ["STRAGGLAR_LL_GENTLE=200"],
}
VARIANTS_HINT = {
    "st_ef": ["STRAGGLAR_STORE_HINT=1"],
    "ld_ef": ["STRAGGLAR_LOAD_HINT=1"],
    "st_ef_ld_ef": ["STRAGGLAR_STORE_HINT=1", "STRAGGLAR_LOAD_HINT=1"],
    "st_el": ["STRAGGLAR_STORE_HINT=2"],
    "ld_el": ["STRAGGLAR_LOAD_HINT=2"],
    "st_el_ld_el": ["STRAGGLAR_STORE_HINT=2", "STRAGGLAR_LOAD_HINT=2"],
}
if "--hint2" in sys.argv:
    VARIANTS_HINT = {k: VARIANTS_HINT[k] for k in ("st_el", "ld_el", "st_el_ld_el")}
VARIANTS_DEFER = {   # round 2 (r02v): the deferred SEND hand-off (since removed) and the scope diagnostics
    "diag_fence_gpu": ["STRAGGLAR_DIAG_FENCE_GPU=1"],
    "diag_acq_gpu": ["STRAGGLAR_DIAG_ACQ_GPU=1"],
}
VARIANTS_HINT3 = {   # round 2: load / store L2 hints again, with the sub-slice-major order
    "ld_ef": ["STRAGGLAR_LOAD_HINT=1"],
    "ld_none": ["STRAGGLAR_LOAD_HINT=0"],
    "st_none": ["STRAGGLAR_STORE_HINT=0"],
    "ld_ef_st_none": ["STRAGGLAR_LOAD_HINT=1", "STRAGGLAR_STORE_HINT=0"],
}
VARIANTS_LIFE = {   # round 2: L2 hints by data lifetime (Op::life), dead data evict_first / no hint
    "life_ef": ["STRAGGLAR_LIFETIME_HINTS=1", "STRAGGLAR_DEAD_HINT=1"],
    "life_none": ["STRAGGLAR_LIFETIME_HINTS=1", "STRAGGLAR_DEAD_HINT=0"],
}
VARIANTS_TUNE3 = {   # round 2: stage ring / CTA shape again, with sub-slice-major order + lifetime hints
    "s4_16k": ["STRAGGLAR_STAGES=4", "STRAGGLAR_STAGE_BYTES=16384"],
    "s3_32k": ["STRAGGLAR_STAGES=3", "STRAGGLAR_STAGE_BYTES=32768"],
    "s4_12k": ["STRAGGLAR_STAGES=4", "STRAGGLAR_STAGE_BYTES=12288"],
    "s2_24k": ["STRAGGLAR_STAGES=2", "STRAGGLAR_STAGE_BYTES=24576"],
    "t512": ["STRAGGLAR_THREADS=512", "STRAGGLAR_MIN_BLOCKS=2"],
    "nolife": ["STRAGGLAR_LIFETIME_HINTS=0"],
}
VARIANTS_TUNE4 = {   # round 2: stage rings around 4 x 12 KB (4 CTAs per SM must still fit)
    "s4_12k": ["STRAGGLAR_STAGES=4", "STRAGGLAR_STAGE_BYTES=12288"],
    "s4_13k": ["STRAGGLAR_STAGES=4", "STRAGGLAR_STAGE_BYTES=13312"],
    "s5_11k": ["STRAGGLAR_STAGES=5", "STRAGGLAR_STAGE_BYTES=11264"],
    "s5_9k": ["STRAGGLAR_STAGES=5", "STRAGGLAR_STAGE_BYTES=9216"],
    "s6_8k": ["STRAGGLAR_STAGES=6", "STRAGGLAR_STAGE_BYTES=8192"],
    "s3_18k": ["STRAGGLAR_STAGES=3", "STRAGGLAR_STAGE_BYTES=18432"],
}
VARIANTS_RS = {   # round 2: Phase A's own stage geometry over the 5 x 11 KB ring
    "s3_16k": ["STRAGGLAR_STAGES=3", "STRAGGLAR_STAGE_BYTES=16384"],
    "rs5": ["STRAGGLAR_RS_STAGES=5"],
    "rs2": ["STRAGGLAR_RS_STAGES=2"],
    "rs4": ["STRAGGLAR_RS_STAGES=4"],
}
VARIANTS_SIG = {"sig": ["STRAGGLAR_SIGNALLER=1"]}   # round 2: signalling warp in Phase B
VARIANTS = (VARIANTS_SIG if "--sig" in sys.argv else VARIANTS_RS if "--rs" in sys.argv else VARIANTS_TUNE4 if "--tune4" in sys.argv else VARIANTS_TUNE3 if "--tune3" in sys.argv else VARIANTS_LIFE if "--life" in sys.argv else VARIANTS_HINT3 if "--hint3" in sys.argv else VARIANTS_DEFER if "--defer" in sys.argv else VARIANTS_LL if "--ll" in sys.argv else VARIANTS_LAG if "--lag" in sys.argv
            else VARIANTS_HINT if ("--hint" in sys.argv or "--hint2" in sys.argv) else VARIANTS_ALL)
os.makedirs(os.path.join(ROOT, "build", "variants"), exist_ok=True)
with ThreadPoolExecutor(4) as ex:
    futs = {k: ex.submit(B.build, True, False, v, os.path.join(ROOT, "build", "variants", f"lib_{k}.so")) for k, v in VARIANTS.items()}
    for k, f in futs.items():
        print(k, f.result())
