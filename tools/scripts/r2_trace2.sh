cd $GRAFT_REPO_ROOT
PPO_EXPERIMENTS=1 PPO_NVCC_EXTRA="-DPPO_TRACE" python paper_1912_06680_b200/build.py > /dev/null 2>&1 || echo build failed
PPO_VARIANT_HEADS=1cta timeout 300 python tools/trace_step.py --B 32 --H 128 --D 256 > gpurun_out/r2_trace2.txt 2>&1
PPO_VARIANT_HEADS=1cta timeout 300 python tools/trace_step.py --B 600 --H 4096 --D 4032 --mhz 1800 >> gpurun_out/r2_trace2.txt 2>&1
python paper_1912_06680_b200/build.py > /dev/null 2>&1
python -c "
import torch; from paper_1912_06680_b200 import _lib as L; print(L.device_info())" >> gpurun_out/r2_trace2.txt 2>&1
echo done
