"""Summarise an ncu report: per-source-line instruction share and stall
reasons (needs -lineinfo builds), grouped by function."""
import collections
import csv
import subprocess
import sys


def load(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    return list(csv.reader(out.splitlines()))


def f(x):
    try:
        return float(x.replace(",", ""))
    except ValueError:
        return 0.0


def main(rep, top=30):
    rows = load(rep)
    agg = collections.OrderedDict()
    hdr = fname = func = None
    for r in rows:
        if r and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r and r[0] == "Function Name":
            func = r[1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if not hdr or len(r) < len(hdr) or not r[0]:
            continue
        key = (fname, int(r[0]), r[1][:70])
        a = agg.setdefault(key, collections.Counter())
        a["inst"] += f(r[7])
        a["stall"] += f(r[4])
        for i, h in enumerate(hdr[32:49]):
            a[h] += f(r[32 + i])
    tot = sum(v["inst"] for v in agg.values()) or 1
    tots = sum(v["stall"] for v in agg.values()) or 1
    print(f"total warp-instructions {tot:.0f}, stall samples {tots:.0f}")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1]["stall"])[:top]:
        st = sorted(((v[h], h[6:]) for h in v if h.startswith("stall_") and v[h] > 0), reverse=True)[:3]
        st = ", ".join(f"{n}:{c:.0f}" for c, n in st)
        print(f"{v['inst'] / tot * 100:5.1f}%i {v['stall'] / tots * 100:5.1f}%s "
              f"{k[0][:14]}:{k[1]:<4} {k[2]:70} {st}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
