"""Kernel shares of the timed steps from an ncu launch list.

    python tools/launch_shares.py LAUNCHES.csv [--steps K] > shares.md

LAUNCHES.csv: `ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file ...
python bench.py --steps K --warmup W ...`.  The last K of the W + K steps are the timed ones: the
list is cut at the `k_update` launches that end each step.  ncu serialises the launches and
flushes caches between them, so only the SHARES are comparable with the bench line.
"""
import argparse
import collections
import csv
import re


def short(name):
    name = re.sub(r"\(.*", "", name)
    name = name.replace("void ", "").replace("kp::", "").replace("<unnamed>::", "")
    return re.sub(r"<.*", "", name).strip()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--steps", type=int, default=2)
    a = ap.parse_args()
    rows = list(csv.reader(open(a.csv)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr, data = rows[hi], rows[hi + 1:]
    kn, mv, mu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    scale = {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0}
    names = [short(r[kn]) for r in data]
    ms = [float(r[mv].replace(",", "")) * scale[r[mu]] for r in data]
    ends = [i for i, n in enumerate(names) if n == "k_update"]
    if len(ends) > a.steps:
        start = ends[-a.steps - 1] + 1
    else:
        start = 0
    end = ends[-1] + 1 if ends else len(names)
    agg = collections.OrderedDict()
    for n, t in zip(names[start:end], ms[start:end]):
        e = agg.setdefault(n, [0, 0.0])
        e[0] += 1
        e[1] += t
    tot = sum(e[1] for e in agg.values())
    print(f"launches {end - start} in the last {min(a.steps, len(ends))} step(s) of {len(names)} listed; "
          f"serialised sum {tot:.1f} ms\n")
    print("| kernel | launches | ms | share |\n|---|---|---|---|")
    for n, e in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        if e[1] / tot < 0.0005:
            continue
        print(f"| `{n}` | {e[0]} | {e[1]:.2f} | {100 * e[1] / tot:.1f}% |")


if __name__ == "__main__":
    main()
