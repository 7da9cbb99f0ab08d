#!/bin/bash
# ncu evidence for one N=1 bench step (run on the GPU box, after the same
# command exited 0 without ncu):  bash tools/profile_step.sh <tag>
# Writes compact summaries only (gpurun_out/ must stay small); the .ncu-rep
# files stay in /tmp on the box.
#   gpurun_out/<tag>_launches.csv     every launch of a 1-step run (durations)
#   gpurun_out/<tag>_ncu_<k>.txt/.json --set full summaries (tools/ncu_summary.py)
set -u
TAG=${1:-r2}
B="bench.py --steps 1 --warmup 1 --no-e2e --no-fp32 --no-c1 --no-cpu"
NCU="ncu --clock-control none"
R=/tmp/ncu_$TAG
mkdir -p gpurun_out $R
timeout 900 $NCU --metrics gpu__time_duration.sum -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv \
  python $B > /dev/null 2>&1
for spec in "lookup:pooled_fwd:1" "bwd:bwd_update:1" "gemm:gemm_kernel:12" "bucket:bucketize:1"; do
  IFS=: read name rx cnt <<< "$spec"
  timeout 1200 $NCU --set full --import-source on -k regex:$rx -c $cnt -f -o $R/$name python $B > /dev/null 2>&1
  python tools/ncu_summary.py $R/$name.ncu-rep "$TAG $name (ncu --set full, tools/profile_step.sh)" \
    --json gpurun_out/${TAG}_ncu_$name.json > gpurun_out/${TAG}_ncu_$name.txt 2>&1
done
ncu -i $R/gemm.ncu-rep --page source --csv --print-source sass 2>/dev/null | head -c 4000000 > $R/gemm_sass.csv
grep -c UTCHMMA $R/gemm_sass.csv > gpurun_out/${TAG}_gemm_sass_counts.txt 2>&1
du -sh gpurun_out
