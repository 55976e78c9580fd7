tag=${1:-x}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/${tag}_bench.log 2>&1
SPHBI_STREAM_CHUNK_LOG2=19 timeout 300 python bench.py --no-cpu-baseline > gpurun_out/${tag}_bench_c19.log 2>&1
SPHBI_STREAM_CHUNK_LOG2=21 timeout 300 python bench.py --no-cpu-baseline > gpurun_out/${tag}_bench_c21.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches.csv python tools/prof_eval.py --reps 2 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_pipe_stub|k_pipe_emit_slots|k_pipe_combine" -c 6 -o gpurun_out/${tag}_full python tools/prof_eval.py --reps 1 > gpurun_out/${tag}_ncu_full.log 2>&1
