"""One-line digest of a bench.py JSON output file (the last line starting with '{')."""
import json
import sys

d = json.loads([ln for ln in open(sys.argv[1]) if ln.startswith("{")][-1])
ks = ("allreduce", "adam", "dp_adam", "wgrad_o", "splitk_reduce", "lstm_fwd_step", "lstm_bwd_step", "wgrad_xh")
print(round(d["value"]), "samples/s", round(d["ms_per_step"], 2), "ms/step", "clock",
      d["clocks"]["sm_mhz"], {k: round(v["ms_per_step"], 3) for k, v in d["kernels"].items()
                              if k in ks})
