"""Build the decode-kernel timing experiments (wrong results, timing only) into scripts/."""
import sys
sys.path.insert(0, ".")
from paper_2410_23918_b200.build import build
for name, flags in [("nosttm", ["-DBS_EXP_NO_STTM"]), ("nomma", ["-DBS_EXP_NO_MMA"]),
                    ("noexpand", ["-DBS_EXP_NO_EXPAND"]), ("nosttm_nomma", ["-DBS_EXP_NO_STTM", "-DBS_EXP_NO_MMA"]),
                    # decode_f8i skeleton (scripts/exp_skeleton.sh)
                    ("skel", ["-DBS_EXP_SKEL"]), ("nosign", ["-DBS_EXP_NOSIGN"]),
                    ("skelns", ["-DBS_EXP_SKEL", "-DBS_EXP_NOSIGN"])]:
    print(build(extra=flags, out=f"/root/repo/scripts/libbitstack_{name}.so"))
