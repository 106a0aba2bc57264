"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv): per kernel the
launch count, mean / total device time and the share of the total (libhap kernels only)."""
import csv
import sys
from collections import defaultdict


def summary(path, skip_first=0):
    rows = [r for r in csv.reader(l for l in open(path) if l.startswith('"'))]
    hdr, rows = rows[0], rows[1:]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[skip_first:]:
        name = r[ki].split("(")[0].replace("void ", "").replace("hap::(anonymous namespace)::", "")
        if not any(k in name for k in ("k1", "k2", "k3")):
            continue
        tot[name] += float(r[vi].replace(",", "")) / 1e3
        cnt[name] += 1
    all_us = sum(tot.values())
    out = []
    for n in sorted(tot, key=lambda n: -tot[n]):
        out.append((n, cnt[n], tot[n] / cnt[n], tot[n], tot[n] / all_us))
    return out


if __name__ == "__main__":
    print(f"{'kernel':40s} {'launches':>8s} {'us/launch':>10s} {'total us':>10s} {'share':>6s}")
    for n, c, m, t, s in summary(sys.argv[1]):
        print(f"{n:40s} {c:8d} {m:10.1f} {t:10.1f} {s:6.3f}")
