#!/bin/bash
# One GPU session of a round (run under gpurun): the GPU test tier, the default
# bench line, the reference arm, and (optionally) the ncu FP64 evidence.
#   bash tools/gpu_round.sh <tag> [tests|notests] [ncu|noncu]
TAG=${1:-rXX}
mkdir -p gpurun_out
if [ "${2:-tests}" = tests ]; then
  python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1
  tail -5 gpurun_out/${TAG}_pytest.log
fi
python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
tail -c 3000 gpurun_out/${TAG}_bench.json
if [ "${3:-noncu}" = ncu ]; then
  bash tools/ncu_fp64_round.sh ${TAG} > gpurun_out/${TAG}_ncu_fp64.log 2>&1
  tail -40 gpurun_out/${TAG}_ncu_fp64.log
fi
