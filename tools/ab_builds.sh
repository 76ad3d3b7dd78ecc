#!/bin/bash
# A/B/... of several builds of libppo5 on ONE box (the boxes differ by +-5% under the power cap).
# Here (with git):   bash tools/ab_builds.sh prep <git-rev-1> <git-rev-2> [<git-rev-3> ...]
#   exports the revisions' sources into .ab/1, .ab/2, ... (git-ignored; they travel with gpurun)
# On the GPU box:    bash tools/ab_builds.sh run [rounds] [bench args...]
#   builds each and runs bench.py with each library in turn (PPO_LIB_PATH), `rounds` times.
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
if [ "$1" = prep ]; then
  shift
  rm -rf $ROOT/.ab; i=1
  for rev in "$@"; do
    mkdir -p $ROOT/.ab/$i
    (cd $ROOT && git archive $rev paper_1912_06680_b200 include | tar -x -C $ROOT/.ab/$i)
    echo "$rev" > $ROOT/.ab/$i/REV
    i=$((i + 1))
  done
  exit 0
fi
ROUNDS=${2:-2}; shift 2 || true
builds=$(ls $ROOT/.ab | sort -n)
for b in $builds; do
  (cd $ROOT/.ab/$b && python paper_1912_06680_b200/build.py > /dev/null 2>&1) || { echo "build $b failed"; exit 1; }
  echo "$b = $(cat $ROOT/.ab/$b/REV)"
done
for i in $(seq 1 $ROUNDS); do
  for b in $builds; do
    PPO_LIB_PATH=$ROOT/.ab/$b/paper_1912_06680_b200/libppo5.so python $ROOT/bench.py --no-e2e --no-cpu-baseline "$@" 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']; print('$b', round(d['value'],1), round(d['ms_per_step'],2), d['clocks']['sm_mhz'], ' '.join(f'{n}={k[n][\"ms_per_step\"]:.2f}' for n in ('lstm_fwd_step','lstm_bwd_step','wgrad_xh','heads_fwd','wgrad_o','loss','adam') if n in k))"
  done
done
