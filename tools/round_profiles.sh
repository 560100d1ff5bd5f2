#!/bin/bash
# The round's committed ncu evidence (run on the GPU box; dev helper):
#  * one ncu --set full capture of the top kernels (CSV exports, no .ncu-rep),
#  * the launch list of one full bench step (gpu__time_duration, cold/serialised).
# Summaries: python tools/summarize_ncu.py kernel|launches ... -> profiles/
R=${1:-r02z}
tools/ncu_capture.sh ${R}_eval_f1 k_evaluate_sep 28 -- python tools/profile_run.py 1 8 1e-3 30
tools/ncu_capture.sh ${R}_eval_f4 k_evaluate_sep 20 -- python tools/profile_run.py 4 8 1e-3 22
tools/ncu_capture.sh ${R}_eval_f6 k_evaluate_sep 38 -- python tools/profile_run.py 6 8 1e-4 40
tools/ncu_capture.sh ${R}_eval_f4_10d k_evaluate_sep 12 -- python tools/profile_run.py 4 10 1e-3 14
tools/ncu_capture.sh ${R}_link_f1 k_link 24 -- python tools/profile_run.py 1 8 1e-3 30
PAGANI_DEFER_BISECT=0 tools/ncu_capture.sh ${R}_split_f1 k_split_bulk 24 -- python tools/profile_run.py 1 8 1e-3 30
tools/ncu_capture.sh ${R}_probe_f6 k_probe_multi 10 -- python tools/profile_run.py 6 8 1e-4 40
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${R}_launches_bench.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline \
  > gpurun_out/${R}_launches_bench.log 2>&1
gzip -f gpurun_out/${R}_launches_bench.csv
ls -la gpurun_out | grep $R
