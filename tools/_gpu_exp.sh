# item-grid strategy experiment + coupling tests
tag=${1:-x}
timeout 600 python -m pytest tests/test_gpu_coupling.py tests/test_gpu_bases.py -x -q > gpurun_out/${tag}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
for g in persist sync 2n; do
  SPHBI_ITEM_GRID=$g timeout 300 python bench.py --no-cpu-baseline > gpurun_out/${tag}_bench_$g.log 2>&1
  SPHBI_ITEM_GRID=$g timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches_$g.csv python tools/prof_eval.py --reps 2 > /dev/null 2>&1
done
