"""Per-launch DRAM traffic, duration and clock of each step kernel from one-launch ncu --set
full captures named gpurun_out/r2_tr_<tag>.ncu-rep -> profiles/r02_traffic.json (read by
bench.py for roofline.traffic), plus a text summary.

    python tools/ncu_traffic2.py profiles/r02_traffic.json gpurun_out/r2_tr_*.ncu-rep"""
import csv
import io
import json
import os
import subprocess
import sys

M = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
     "sm__cycles_elapsed.avg.per_second", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
     "lts__t_sectors_srcunit_tex.sum", "lts__t_sectors_srcunit_ltcfabric.sum",
     "smsp__inst_executed.sum", "launch__registers_per_thread"]
SCALE = {"Ghz": 1e9, "Mhz": 1e6, "hz": 1.0, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1e-9,
         "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}


def main(dst, reps):
    out = {"source": "ncu --set full --clock-control none, one launch per kernel class, "
                     "tools/profile_step.py --B 38400 (round-2 tree)", "kernels": {}}
    lines = []
    for p in reps:
        tag = os.path.basename(p).split("_tr_", 1)[1][:-len(".ncu-rep")]
        txt = subprocess.run(["ncu", "-i", p, "--page", "raw", "--csv", "--metrics", ",".join(M)],
                             capture_output=True, text=True).stdout
        r = list(csv.reader(io.StringIO(txt)))
        if len(r) < 3:
            continue
        hdr, units, row = r[0], r[1], r[2]
        v = {}
        for m in M:
            if m in hdr:
                i = hdr.index(m)
                try:
                    v[m] = float(row[i].replace(",", "")) * SCALE.get(units[i], 1.0)
                except ValueError:
                    pass
        traffic = v.get("dram__bytes_read.sum", 0) + v.get("dram__bytes_write.sum", 0)
        out["kernels"][tag] = {"dram_bytes_per_launch": traffic,
                               "dram_read_bytes": v.get("dram__bytes_read.sum"),
                               "ncu_seconds_per_launch": v.get("gpu__time_duration.sum"),
                               "sm_clock_hz": v.get("sm__cycles_elapsed.avg.per_second"),
                               "tensor_active_pct": v.get(M[4]),
                               "l2_sectors_from_sm": v.get(M[5]),
                               "l2_sectors_cross_die": v.get(M[6]),
                               "warp_instructions": v.get(M[7]),
                               "kernel": row[hdr.index("Kernel Name")][:120]}
        k = out["kernels"][tag]
        lines.append(f"{tag:14s} {k['ncu_seconds_per_launch'] * 1e3 if k['ncu_seconds_per_launch'] else 0:9.3f} ms  "
                     f"DRAM {traffic / 1e9:8.3f} GB  clock {(k['sm_clock_hz'] or 0) / 1e9:5.2f} GHz  "
                     f"tensor {k['tensor_active_pct'] or 0:5.1f}%  L2<-SM {(k['l2_sectors_from_sm'] or 0) * 32 / 1e9:7.2f} GB  "
                     f"cross-die {(k['l2_sectors_cross_die'] or 0) * 32 / 1e9:6.2f} GB")
    with open(dst, "w") as f:
        json.dump(out, f, indent=1)
    with open(dst.replace(".json", ".txt"), "w") as f:
        f.write(out["source"] + "\n" + "\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2:])
