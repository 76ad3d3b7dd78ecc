#!/bin/bash
# A/B two builds of libppo5 on ONE box (the boxes differ by +-5% under the power cap):
#   bash tools/ab_builds.sh <git-rev-A> <git-rev-B> [rounds] [bench args...]
# Rev A and B are built into /tmp worktrees; bench.py runs alternately with each library.
set -e
A=$1; B=$2; ROUNDS=${3:-2}; shift 3 || true
ROOT=$(cd "$(dirname "$0")/.." && pwd)
for r in A B; do
  rev=$([ $r = A ] && echo $A || echo $B)
  d=/tmp/ab_$r
  rm -rf $d; mkdir -p $d
  (cd $ROOT && git archive $rev paper_1912_06680_b200 include | tar -x -C $d)
  (cd $d && python paper_1912_06680_b200/build.py > /dev/null 2>&1) || { echo "build $r failed"; exit 1; }
done
for i in $(seq 1 $ROUNDS); do
  for r in A B; do
    PPO_LIB_PATH=/tmp/ab_$r/paper_1912_06680_b200/libppo5.so python $ROOT/bench.py --no-e2e --no-cpu-baseline "$@" 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']; print('$r', round(d['value'],1), round(d['ms_per_step'],2), d['clocks']['sm_mhz'], ' '.join(f'{n}={k[n][\"ms_per_step\"]:.2f}' for n in ('lstm_fwd_step','lstm_bwd_step','wgrad_xh','heads_fwd','wgrad_o','loss','adam') if n in k))"
  done
done
