# GPU iteration: gpu tests, bench, and the cfg2 launch list (ncu timing only)
tag=${1:-x}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
timeout 400 python bench.py --no-cpu-baseline > gpurun_out/${tag}_bench.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches.csv python tools/prof_eval.py --reps 2 > gpurun_out/${tag}_ncu.log 2>&1
