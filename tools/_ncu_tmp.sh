ncu --set full --clock-control none --import-source on -k regex:"k_pipe_emit_slots|k_pipe_combine|k_pre_class" -c 3 -o gpurun_out/s1_full python tools/prof_eval.py --reps 1 > gpurun_out/s1_ncu.log 2>&1
ls -la gpurun_out
