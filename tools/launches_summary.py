"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list per kernel (share of
device time).  ncu times are cold-cache and serialised: compare shares, not absolutes."""
import collections
import csv
import io
import sys


def load(path):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    return list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))


def main(path, tag_filter=None):
    rows = load(path)
    scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3,
             "ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}
    agg = collections.OrderedDict()
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0].replace("void ", "")
        v = float(r["Metric Value"].replace(",", "")) * scale[r["Metric Unit"]]
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
    mine = {k: v for k, v in agg.items() if "ppo::" in k or "tc_gemm" in k}
    tot_all = sum(v[1] for v in agg.values())
    tot = sum(v[1] for v in mine.values())
    print(f"{len(rows)} launches total; libppo5 kernels {sum(v[0] for v in mine.values())} "
          f"launches, {tot:.1f} ms of {tot_all:.1f} ms device time")
    print(f"{'kernel':84s} {'launches':>8s} {'ms':>10s} {'share(libppo5)':>15s}")
    for k, (n, ms) in sorted(mine.items(), key=lambda kv: -kv[1][1]):
        print(f"{k[:84]:84s} {n:8d} {ms:10.3f} {ms / tot:15.3f}")


if __name__ == "__main__":
    main(sys.argv[1])
