#!/bin/bash
# One ncu --set full capture of a kernel, exported to CSVs on the GPU box
# (the .ncu-rep itself is too large to bring back).  Dev helper.
#   tools/ncu_capture.sh LABEL KERNEL_REGEX SKIP -- python tools/profile_run.py ...
set -u
LABEL=$1; KRE=$2; SKIP=$3; shift 4
OUT=gpurun_out/$LABEL
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:$KRE" -s "$SKIP" -c 1 \
  -o "/tmp/$LABEL" "$@" > "$OUT.log" 2>&1
ncu -i "/tmp/$LABEL.ncu-rep" --page raw --csv > "$OUT.raw.csv" 2>/dev/null
ncu -i "/tmp/$LABEL.ncu-rep" --page details --csv > "$OUT.details.csv" 2>/dev/null
ncu -i "/tmp/$LABEL.ncu-rep" --page source --csv --print-source sass > "$OUT.sass.csv" 2>/dev/null
ncu -i "/tmp/$LABEL.ncu-rep" --page source --csv --print-source cuda > "$OUT.cuda.csv" 2>/dev/null
gzip -f "$OUT.sass.csv" "$OUT.cuda.csv"
rm -f "/tmp/$LABEL.ncu-rep"
ls -la "$OUT".*
