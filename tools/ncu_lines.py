"""Per-source-line executed instructions and stall samples of one kernel in an ncu report
(--set full --import-source on), normalised per unit:  python tools/ncu_lines.py REP UNITS [N]"""
import collections
import csv
import subprocess
import sys

rep, units = sys.argv[1], float(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 50
txt_csv = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
agg, st, txt = collections.Counter(), collections.Counter(), {}
cur, hdr = None, None


def num(x):
    try:
        return int(x)
    except ValueError:
        return 0


for r in csv.reader(txt_csv.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        i_ex = hdr.index("Instructions Executed")
        i_st = hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None or len(r) <= i_ex or not r[0].isdigit():
        continue
    k = (cur, int(r[0]))
    agg[k] += num(r[i_ex])
    st[k] += num(r[i_st])
    txt[k] = r[1][:90]
tot, S = sum(agg.values()), max(1, sum(st.values()))
print(f"instructions per unit {tot / units:.1f}; stall samples {S}")
for k, n in agg.most_common(top):
    print(f"{n / units:7.1f} {100 * st[k] / S:5.1f}% {k[0]}:{k[1]:<5d} {txt[k]}")
