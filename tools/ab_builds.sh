#!/bin/bash
# A/B two builds of libppo5 on ONE box (the boxes differ by +-5% under the power cap).
# Here (with git):   bash tools/ab_builds.sh prep <git-rev-A> <git-rev-B>
#   exports both revisions' sources into .ab/A and .ab/B (git-ignored; they travel with gpurun)
# On the GPU box:    bash tools/ab_builds.sh run [rounds] [bench args...]
#   builds both and runs bench.py alternately with each library (PPO_LIB_PATH).
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
if [ "$1" = prep ]; then
  for r in A B; do
    rev=$([ $r = A ] && echo $2 || echo $3)
    rm -rf $ROOT/.ab/$r; mkdir -p $ROOT/.ab/$r
    (cd $ROOT && git archive $rev paper_1912_06680_b200 include | tar -x -C $ROOT/.ab/$r)
    echo "$rev" > $ROOT/.ab/$r/REV
  done
  exit 0
fi
ROUNDS=${2:-2}; shift 2 || true
for r in A B; do
  (cd $ROOT/.ab/$r && python paper_1912_06680_b200/build.py > /dev/null 2>&1) || { echo "build $r failed"; exit 1; }
done
echo "A = $(cat $ROOT/.ab/A/REV)  B = $(cat $ROOT/.ab/B/REV)"
for i in $(seq 1 $ROUNDS); do
  for r in A B; do
    PPO_LIB_PATH=$ROOT/.ab/$r/paper_1912_06680_b200/libppo5.so python $ROOT/bench.py --no-e2e --no-cpu-baseline "$@" 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']; print('$r', round(d['value'],1), round(d['ms_per_step'],2), d['clocks']['sm_mhz'], ' '.join(f'{n}={k[n][\"ms_per_step\"]:.2f}' for n in ('lstm_fwd_step','lstm_bwd_step','wgrad_xh','heads_fwd','wgrad_o','loss','adam') if n in k))"
  done
done
