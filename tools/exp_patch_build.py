"""Experiment-only builds: copy csrc/ to a scratch directory, apply a named source patch to the
GEMM and build tools/exp/libsplit3_<tag>.so (the product sources stay untouched).  Used with
tools/power_ab.py (EXP_LIB) to measure what a change would buy before building it properly.

  python tools/exp_patch_build.py TAG       TAG in PATCHES

Patches (results of these builds are WRONG by design; they time the machine, not the method):
  nob    the producer loads B's planes only for the first STAGES k-blocks of each CTA, then reuses
         whatever the stage holds: the GEMM without B's L2->SMEM traffic (upper bound of what TMA
         multicast of B over a cluster of pairs could save);
  halfb  B's planes loaded on every other k-block only (models a 2-pair cluster sharing B);
  halfab both A's and B's planes on every other k-block (models a 2 x 2 cluster of pairs);
  dupab  every odd k-block re-loads the previous k-block's A and B tiles (L2 hits): DRAM traffic
         halves, L2->SMEM traffic unchanged (separates the two in the A/B above).
"""
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2011_11188_b200 import _build  # noqa: E402

ANCHOR_TX = "                    if (leader) mbar_expect_tx(fb, TX_BYTES);\n"
ANCHOR_A1 = "                    load_a(0, &mapA1);\n                    if (!FB) load_b(B_OFF, &mapB1);\n"
ANCHOR_LO = ("                        load_a(TILE_A_BYTES, &mapA2);\n"
             "                        if (!FB) load_b(B_OFF + TILE_B_BYTES, &mapB2);\n")
ANCHOR_ADV = "                __syncwarp();\n                if (++stage == STAGES) { stage = 0; phase ^= 1; }\n            }\n        }\n    } else if (warp == 1) {"
ANCHOR_DECL = "        int64_t idx = 0;\n        for (int64_t unit = pair; unit < num_units; unit += num_pairs, idx++) {"


ANCHOR_X = "                const int32_t x = kb * BK;\n"


def patch(src: str, skip_a: str, skip_b: str, dup: bool = False) -> str:
    if dup:
        assert src.count(ANCHOR_X) == 1
        src = src.replace(ANCHOR_X, "                const int32_t x = ((kb > kb_begin && ((kb - kb_begin) & 1)) ? kb - 1 : kb) * BK;\n")
    for a in (ANCHOR_TX, ANCHOR_A1, ANCHOR_LO, ANCHOR_ADV, ANCHOR_DECL):
        assert src.count(a) == 1, a
    src = src.replace(ANCHOR_DECL, "        int64_t idx = 0;\n        int64_t gkb = 0;\n"
                      "        for (int64_t unit = pair; unit < num_units; unit += num_pairs, idx++) {")
    src = src.replace(ANCHOR_TX,
                      f"                    const bool skip_a = gkb >= STAGES && ({skip_a});\n"
                      f"                    const bool skip_b = gkb >= STAGES && ({skip_b});\n"
                      "                    if (leader) mbar_expect_tx(fb, TX_BYTES - (skip_a ? 2u * 2u * TILE_A_BYTES : 0u)"
                      " - (skip_b ? 2u * 2u * TILE_B_BYTES : 0u));\n")
    src = src.replace(ANCHOR_A1, "                    if (!skip_a) load_a(0, &mapA1);\n"
                                 "                    if (!FB && !skip_b) load_b(B_OFF, &mapB1);\n")
    src = src.replace(ANCHOR_LO, "                        if (!skip_a) load_a(TILE_A_BYTES, &mapA2);\n"
                                 "                        if (!FB && !skip_b) load_b(B_OFF + TILE_B_BYTES, &mapB2);\n")
    src = src.replace(ANCHOR_ADV, "                __syncwarp();\n                gkb++;\n"
                                  "                if (++stage == STAGES) { stage = 0; phase ^= 1; }\n            }\n        }\n"
                                  "    } else if (warp == 1) {")
    return src


PATCHES = {
    "nob": ("false", "true"),
    "halfb": ("false", "(gkb & 1) != 0"),
    "halfab": ("(gkb & 1) != 0", "(gkb & 1) != 0"),
    "dupab": ("false", "false", True),
}

if __name__ == "__main__":
    tag = sys.argv[1]
    skip_a, skip_b, *dup = PATCHES[tag]
    tmp = tempfile.mkdtemp()
    csrc = os.path.join(tmp, "pkg", "csrc")          # csrc/ includes ../../include/split3.h
    shutil.copytree(_build.CSRC, csrc)
    shutil.copytree(os.path.join(ROOT, "include"), os.path.join(tmp, "include"))
    g = os.path.join(csrc, "gemm3.cu")
    with open(g) as f:
        s = f.read()
    with open(g, "w") as f:
        f.write(patch(s, skip_a, skip_b, bool(dup and dup[0])))
    out = os.path.join(ROOT, "tools", "exp", f"libsplit3_{tag}.so")
    cmd = [_build.NVCC, *_build.NVCC_FLAGS, "-shared", "-o", out,
           *sorted(os.path.join(csrc, x) for x in os.listdir(csrc) if x.endswith(".cu")),
           "-I", os.path.join(ROOT, "include")]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        print(r.stderr[-3000:])
        sys.exit(1)
    print(out)
