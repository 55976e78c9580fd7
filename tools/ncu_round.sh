# ncu evidence for the round (run under gpurun; results land in gpurun_out/):
# launch list of the bench command, --set full of the K4 pipeline kernels on
# the cfg2 workload, the P3 (cfg4) launch list + full capture of its stub
# kernel, and the cfg3 launch list (pair finding).
set -x
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 > gpurun_out/ncu_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_pipe_stub|k_pipe_emit_slots|k_pipe_combine|k_pre_class|k_sig_scatter" -c 8 -o gpurun_out/pipe_full python tools/prof_eval.py --reps 1 > gpurun_out/ncu_full.log 2>&1
REPS=1 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg4.csv python tools/cfg4_time.py > gpurun_out/ncu_cfg4.log 2>&1
REPS=1 ncu --set full --clock-control none --import-source on -k regex:"k_p3_stub|k_p3_combine" -c 2 -o gpurun_out/p3_full python tools/cfg4_time.py > gpurun_out/ncu_p3.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg3.csv python tools/prof_eval.py --config cfg3 --reps 1 > gpurun_out/ncu_cfg3.log 2>&1
ls -la gpurun_out
