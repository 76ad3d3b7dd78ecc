"""Build libppo5.so in-tree with nvcc for sm_100a (no JIT, no torch extension machinery)."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libppo5.so")
SOURCES = ["api.cu", "kernels.cu", "tc_path.cu", "comm.cu", "buffer.cu", "infer.cu", "aux.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def _nccl_dir():
    """NCCL bundled with torch (2.28.x): link the same library torch loads, so one NCCL
    lives in the process (the system 2.27 lacks symbols torch needs)."""
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    for base in (spec.submodule_search_locations or []) if spec else []:
        d = os.path.join(base, "nccl")
        if os.path.exists(os.path.join(d, "lib", "libnccl.so.2")):
            return d
    return None


_NCCL = _nccl_dir()
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xptxas", "-v", "-I" + os.path.join(ROOT, "include")]
if _NCCL:
    FLAGS.append("-I" + os.path.join(_NCCL, "include"))
# A/B timing builds only: PPO_EXPERIMENTS=1 compiles in the PPO_* environment overrides
# (common.cuh knob()); a release build reads no environment variable
if os.environ.get("PPO_EXPERIMENTS", "0") not in ("", "0"):
    FLAGS.append("-DPPO_EXPERIMENTS")
# extra nvcc flags for experiment builds (e.g. -DPPO_SUSPEND_HINT_NS=2000)
FLAGS += os.environ.get("PPO_NVCC_EXTRA", "").split()
STAMP = os.path.join(CSRC, ".build_flags")


def _stale(obj, deps):
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, jobs: int = 4) -> str:
    flags = " ".join(FLAGS)
    if not os.path.exists(STAMP) or open(STAMP).read() != flags:
        # other flags than the last build (e.g. an experiments build): rebuild everything
        for f in os.listdir(CSRC):
            if f.endswith(".o"):
                os.remove(os.path.join(CSRC, f))
        if os.path.exists(OUT):
            os.remove(OUT)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    headers.append(os.path.join(ROOT, "include", "ppo5.h"))
    objs, procs = [], []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(CSRC, src[:-3] + ".o")
        objs.append(o)
        if _stale(o, [s] + headers):
            cmd = [NVCC, *FLAGS, "-c", s, "-o", o]
            procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
    for src, p in procs:
        out, _ = p.communicate()
        log = out.decode()
        with open(os.path.join(CSRC, src[:-3] + ".ptxas.log"), "w") as f:
            f.write(log)
        if p.returncode != 0:
            sys.stderr.write(log)
            raise RuntimeError(f"nvcc failed on {src}")
        if verbose:
            sys.stdout.write(log)
    if _stale(OUT, objs):
        if _NCCL:
            libdir = os.path.join(_NCCL, "lib")
            link = ["-L" + libdir, "-l:libnccl.so.2", "-Xlinker", "-rpath," + libdir]
        else:
            link = ["-lnccl"]
        cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", OUT, *objs,
               *link]
        subprocess.run(cmd, check=True)
    with open(STAMP, "w") as f:
        f.write(flags)
    return OUT


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
