"""Per-launch DRAM traffic and duration of each libppo5 kernel class from ncu --set full
reports -> profiles/<name>.json, read by bench.py for roofline.traffic.

    python tools/ncu_traffic.py out.json rep1.ncu-rep rep2.ncu-rep ..."""
import csv
import io
import json
import subprocess
import sys

# kernel-name fragment -> bench kernel tag (first match wins)
TAGS = [("EpiLstmFwd", "lstm_fwd_step"), ("EpiLstmBwd", "lstm_bwd_step"),
        ("tc_gemm2_kernel<1, 1, 4, 2", "wgrad_xh"), ("tc_gemm_kernel<224", "heads_fwd"),
        ("tc_gemm_kernel<256, 1, 1", "wgrad_o"), ("pack_x", "pack_x"), ("loss_kernel", "loss"),
        ("adam_kernel", "adam"), ("gae_kernel", "gae"), ("gae_long", "gae")]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
        "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}


def rows(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    return r[0], r[1], r[2:]


def main(dst, paths):
    agg = {}
    for p in paths:
        hdr, units, data = rows(p)
        ix = {h: i for i, h in enumerate(hdr)}
        for row in data:
            name = row[ix["Kernel Name"]]
            tag = next((t for frag, t in TAGS if frag in name), None)
            if tag is None:
                continue
            def val(k):
                v = row[ix[k]].replace(",", "")
                try:
                    return float(v) * UNIT.get(units[ix[k]], 1.0)
                except ValueError:
                    return None
            rd, wr, dur = val("dram__bytes_read.sum"), val("dram__bytes_write.sum"), val("gpu__time_duration.sum")
            if rd is None or wr is None:
                continue
            a = agg.setdefault(tag, {"launches_captured": 0, "dram_bytes": 0.0, "seconds": 0.0})
            a["launches_captured"] += 1
            a["dram_bytes"] += rd + wr
            a["seconds"] += dur or 0.0
    res = {t: {"dram_bytes_per_launch": a["dram_bytes"] / a["launches_captured"],
               "ncu_seconds_per_launch": a["seconds"] / a["launches_captured"],
               "launches_captured": a["launches_captured"]} for t, a in agg.items()}
    json.dump({"source": "ncu --set full --clock-control none, tools/profile_step.py --B 38400",
               "reports": paths, "kernels": res}, open(dst, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2:])
