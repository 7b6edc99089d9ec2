"""Per-kernel SASS opcode histogram of the built library (no GPU needed).

    python tools/sass_histogram.py > profiles/r02_sass_histogram.md

Disassembles paper_2405_15603_b200/libkfac_pinn_b200.so with cuobjdump -sass and counts, per
kernel, the instructions that prove the FP64 tensor-core / tcgen05 / TMA / cluster paths: DMMA
(mma.sync .f64), UTCIMMA (tcgen05.mma kind::i8), LDTM (tcgen05.ld from TMEM), UTCBAR
(tcgen05.commit), FFMA2 (packed f32x2 FMA), UTMALDG (TMA tensor loads), UBLKCP (bulk copies), SYNCS (mbarrier
arrive/wait), DFMA, LDGSTS (cp.async), UCGABAR (cluster barrier arrive/wait), BAR (CTA
barrier), and the total instruction count.
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2405_15603_b200", "libkfac_pinn_b200.so")
OPS = ("DMMA", "UTCIMMA", "LDTM", "UTMALDG", "UTCBAR", "UBLKCP", "SYNCS", "DFMA", "FFMA2", "LDGSTS",
       "UCGABAR", "BAR")


def demangle(names):
    try:
        out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True,
                             check=True).stdout.splitlines()
        return dict(zip(names, out))
    except (OSError, subprocess.CalledProcessError):
        return {n: n for n in names}


def main():
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True,
                          check=True).stdout
    hist = collections.OrderedDict()
    cur = None
    for line in sass.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            hist[cur] = collections.Counter()
            continue
        if cur is None:
            continue
        m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[\w.]+)?", line)
        if m:
            op = m.group(1)
            hist[cur]["total"] += 1
            for k in OPS:
                if op == k or op.startswith(k + ".") or (k == "UCGABAR" and op.startswith(k)):
                    hist[cur][k] += 1
    names = demangle(list(hist))
    print("# SASS opcode histogram, libkfac_pinn_b200.so (sm_100a)\n")
    print("`python tools/sass_histogram.py` (cuobjdump -sass).  Template instances of one "
          "kernel are summed.\n")
    agg = collections.OrderedDict()
    for mangled, cnt in hist.items():
        name = names[mangled]
        base = name.replace("(anonymous namespace)::", "")
        base = re.sub(r"^void ", "", base)
        base = re.split(r"[<(]", base)[0].split("::")[-1]
        a = agg.setdefault(base, collections.Counter())
        a.update(cnt)
        a["instances"] += 1
    cols = ("instances", "total") + OPS
    print("| kernel | " + " | ".join(cols) + " |")
    print("|---|" + "---|" * len(cols))
    for k, c in sorted(agg.items(), key=lambda kv: -kv[1]["DMMA"]):
        print(f"| `{k}` | " + " | ".join(str(c.get(x, 0)) for x in cols) + " |")


if __name__ == "__main__":
    sys.exit(main())
