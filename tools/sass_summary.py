"""SASS evidence for the hot kernels: per-kernel counts of the tensor-core,
TMEM, bulk-copy and barrier instructions, plus a short excerpt around the
first tensor-core MMA.  Reads the in-tree library (no GPU needed).

    python tools/sass_summary.py [OUT_TXT]      (default profiles/r02/sass_summary.txt)
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2406_10938_b200", "libdetlsh_b200.so")
KERNELS = ["project_tc_kernel", "tc_score_kernel", "project_dmma_kernel", "query_fast_kernel", "proj_tc_fixup_kernel",
           "tc_finish_f32_kernel"]
OPS = ["UTCIMMA", "UTCHMMA", "UTCQMMA", "UTCBAR", "LDTM", "UTMALDG", "UBLKCP", "SYNCS", "DMMA", "DFMA", "IDP",
       "HMMA", "BAR", "ATOMS", "ATOMG", "RED", "I2F", "F2F", "LDG", "STG", "LDS", "STS"]


def main(out):
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
    funcs = re.split(r"\n\s*Function : ", sass)[1:]
    lines = [f"# SASS summary of {os.path.relpath(LIB, ROOT)} (cuobjdump -sass; sm_100a)", ""]
    for f in funcs:
        name = f.split("\n", 1)[0].strip()
        short = next((k for k in KERNELS if k in name), None)
        if short is None:
            continue
        m = re.search(r"ILi(\d+)ELi(\d+)ELb(\d)E|ILi(\d+)ELb(\d)E", name)
        tag = short + (f"<{','.join(g for g in m.groups() if g is not None)}>" if m else "")
        body = [ln for ln in f.split("\n") if re.match(r"\s*/\*[0-9a-f]{4,}\*/", ln)]
        cnt = collections.Counter()
        first_mma = None
        for i, ln in enumerate(body):
            ins = re.sub(r"^\s*/\*[0-9a-f]+\*/\s*(@!?U?P\w+\s+)?", "", ln).split(" ")[0]
            base = ins.split(".")[0]
            if base in OPS:
                cnt[base] += 1
            if first_mma is None and base in ("UTCIMMA", "UTCHMMA", "UTCQMMA", "DMMA"):
                first_mma = i
        lines.append(f"{tag}: {len(body)} instructions; " + ", ".join(f"{k}={cnt[k]}" for k in OPS if cnt[k]))
        if first_mma is not None:
            lines.append("  excerpt around the first MMA:")
            for ln in body[max(0, first_mma - 4):first_mma + 5]:
                lines.append("    " + re.sub(r"\s+", " ", ln.strip())[:140])
        lines.append("")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    with open(out, "w") as fh:
        fh.write("\n".join(lines))
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "r02", "sass_summary.txt"))
