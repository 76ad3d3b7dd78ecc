"""Summarise ncu --set full reports (raw page) into a short text table for profiles/."""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "sm clock"),
    ("sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed",
     "tcgen05 bf16 MMA % of peak (elapsed)"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe active %"),
    ("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
     "tensor pipe active (realtime) %"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram throughput %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("smsp__average_warp_latency_issue_stalled_long_scoreboard", "stall long_scoreboard"),
]


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def main(paths):
    for p in paths:
        hdr, units, data = raw(p)
        idx = {h: i for i, h in enumerate(hdr)}
        for row in data:
            print(f"== {p}")
            print(f"   kernel: {row[idx['Kernel Name']][:110]}")
            for key, label in KEYS:
                if key in idx:
                    print(f"   {label:38s} {row[idx[key]]:>16s} {units[idx[key]]}")
            if "dram__bytes_read.sum" in idx:
                def tob(v, u):
                    f = float(v.replace(",", ""))
                    return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
                r = tob(row[idx["dram__bytes_read.sum"]], units[idx["dram__bytes_read.sum"]])
                w = tob(row[idx["dram__bytes_write.sum"]], units[idx["dram__bytes_write.sum"]])
                print(f"   {'dram traffic (read+write)':38s} {(r + w) / 1e9:16.3f} GB")


if __name__ == "__main__":
    main(sys.argv[1:])
