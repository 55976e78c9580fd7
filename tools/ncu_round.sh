set -x
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 > gpurun_out/ncu_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_pipe_stub|k_pipe_emit|k_pipe_count|k_pipe_combine" -c 4 -o gpurun_out/pipe_full python tools/prof_eval.py --reps 1 > gpurun_out/ncu_full.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_find|k_p3" -c 3 -o gpurun_out/p3_full python tools/cfg4_time.py > gpurun_out/ncu_p3.log 2>&1
ls -la gpurun_out
