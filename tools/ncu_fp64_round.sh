#!/bin/bash
# FP64 roofline evidence of the K4 pipeline kernels (run under gpurun, one GPU):
# ncu instruction counts / FP64-pipe % / DRAM bytes on the cfg5 workload (first
# 1M particles of the scene: a uniform sample, ~11M pairs) and on cfg2 mode A,
# parsed into gpurun_out/<tag>_fp64_<workload>.{csv,json,_summary.txt}.
#   bash tools/ncu_fp64_round.sh <tag> [precision]
set -x
TAG=${1:-r02m}
export SPHBI_PRECISION=${2:-auto}
M=$(python -c "import sys; sys.path.insert(0,'tools'); import ncu_fp64; print(','.join(ncu_fp64.METRICS))")
mkdir -p gpurun_out
for W in cfg5 cfg2a; do
  EXTRA=""
  [ "$W" = cfg5 ] && EXTRA="--particles 1000000"
  python tools/prof_target.py $W $EXTRA > gpurun_out/${TAG}_target_$W.json 2> gpurun_out/${TAG}_target_$W.err || exit 1
  ncu --metrics $M --clock-control none --csv --log-file gpurun_out/${TAG}_fp64_$W.csv \
      python tools/prof_target.py $W $EXTRA > gpurun_out/${TAG}_ncu_$W.log 2>&1
  PAIRS=$(python -c "import json; print(json.loads(open('gpurun_out/${TAG}_target_$W.json').readline())['pairs'])")
  python tools/ncu_fp64.py parse gpurun_out/${TAG}_fp64_$W.csv $PAIRS gpurun_out/${TAG}_fp64_$W.json "$W precision=$SPHBI_PRECISION" \
      > gpurun_out/${TAG}_fp64_${W}_summary.txt 2>&1
  cat gpurun_out/${TAG}_fp64_${W}_summary.txt
done
