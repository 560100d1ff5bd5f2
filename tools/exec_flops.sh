#!/bin/bash
# Executed FP64 operations of k_evaluate (ncu SASS op counters) per integrand,
# over every k_evaluate launch of a 12-iteration 8D run (dev helper; the
# output feeds profiles/r02_executed_flops.json via tools/exec_flops.py).
mkdir -p gpurun_out
for f in 1 2 3 4 5 6; do
  timeout 900 ncu --metrics smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,gpu__time_duration.sum \
    --clock-control none -k regex:k_evaluate_sep --csv --log-file gpurun_out/r02_execflops_f$f.csv \
    python tools/profile_run.py $f 8 1e-3 12 > gpurun_out/r02_execflops_f$f.log 2>&1
done
