"""Build timing-experiment variants of libbitstack.so (wrong values, timing only) into
scripts/variants/lib_<name>.so; scripts/run_variants.sh swaps each in and runs bench.py."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2410_23918_b200 import build as B  # noqa: E402

VARIANTS = {
    "base": [],
    "occ2": ["-DBS_MX_R1=2", "-DBS_MX_OCC1=2"],
    "occ2r1": ["-DBS_MX_R1=1", "-DBS_MX_OCC1=2"],
    "occ2skel": ["-DBS_MX_R1=2", "-DBS_MX_OCC1=2", "-DBS_MX_EXP_NOST", "-DBS_MX_EXP_NOMMA", "-DBS_MX_EXP_NOEXP"],
    "r2s6": ["-DBS_MX_R1=2", "-DBS_MX_NSLOT=6"],
    "r1s8": ["-DBS_MX_R1=1", "-DBS_MX_NSLOT=8"],
    "r1s12": ["-DBS_MX_R1=1", "-DBS_MX_NSLOT=12"],
    "r2s4": ["-DBS_MX_R1=2"],
    "st4": ["-DBS_MX_STAGES=4"],
    "st6": ["-DBS_MX_STAGES=6"],
    "st12": ["-DBS_MX_STAGES=12"],
    "rg32": ["-DBS_RG_COLS=32"],
    "rgbar": ["-DBS_RG_BARSYNC"],
    "rgsame": ["-DBS_RG_SAMESMSP"],
    "rgspinfast": ["-DBS_RG_SPIN_FAST"],
    "rghv1": ["-DBS_RG_HALVES=1", "-DBS_RG_MMA2=0"],
    "rgmma1": ["-DBS_RG_MMA2=0"],
    "sl20k": ["-DBS_SLEEP_NS=20000u"],
    "sl1k": ["-DBS_SLEEP_NS=1000u"],
    "sl200": ["-DBS_SLEEP_NS=200u"],
    "rghv4": ["-DBS_RG_HALVES=4"],
    "rg32same": ["-DBS_RG_COLS=32", "-DBS_RG_SAMESMSP"],
    "rgspin": ["-DBS_RG_SPIN"],
    "rgnoapply": ["-DBS_RG_EXP_NOAPPLY"],
    "rgnocopy": ["-DBS_RG_EXP_NOCOPY"],
    "rgnoboth": ["-DBS_RG_EXP_NOAPPLY", "-DBS_RG_EXP_NOCOPY"],
    "skel": ["-DBS_MX_EXP_NOST", "-DBS_MX_EXP_NOMMA", "-DBS_MX_EXP_NOEXP"],
}
if __name__ == "__main__":
    names = sys.argv[1:] or list(VARIANTS)
    os.makedirs(os.path.join(ROOT, "scripts", "variants"), exist_ok=True)
    for n in names:
        out = os.path.join(ROOT, "scripts", "variants", f"lib_{n}.so")
        B.build(force=True, extra=VARIANTS[n], out=out)
        print(out)
