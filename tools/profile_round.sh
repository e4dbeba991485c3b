#!/bin/bash
# Round profile capture (run under gpurun, one GPU).  Each command first runs
# plainly and must exit 0 before it is repeated under ncu.
#   1. launch list of the bench command (cold-cache, serialised: use SHARES)
#   2. ncu --set full of the C3 kernels (column passes, fused product rows)
#      and of the C4 Goldilocks passes
set -u
R=${1:-r02}
mkdir -p gpurun_out
BENCH="python bench.py --steps 2 --warmup 3 --no-extras --no-cpu-baseline"
$BENCH > gpurun_out/${R}_bench_plain.json 2> gpurun_out/${R}_bench_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${R}_launches.csv $BENCH > gpurun_out/${R}_ncu_launches.log 2>&1
echo launches_rc=$?
python tools/prof_run.py c3 > gpurun_out/${R}_plain_c3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:k_col|k_row" -s 4 -c 4 \
    -o gpurun_out/${R}_full_c3 python tools/prof_run.py c3 > gpurun_out/${R}_ncu_full_c3.log 2>&1
echo full_c3_rc=$?
python tools/prof_run.py c4 > gpurun_out/${R}_plain_c4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:k_gcols|k_grows|k_cols|k_rows" -s 2 -c 2 \
    -o gpurun_out/${R}_full_c4 python tools/prof_run.py c4 > gpurun_out/${R}_ncu_full_c4.log 2>&1
echo full_c4_rc=$?
python tools/prof_run.py c5 > gpurun_out/${R}_plain_c5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:k_gcols|k_gpmul|k_cols|k_rows|k_carry" -s 7 -c 7 \
    -o gpurun_out/${R}_full_c5 python tools/prof_run.py c5 > gpurun_out/${R}_ncu_full_c5.log 2>&1
echo full_c5_rc=$?
python tools/ncu_summary.py launches gpurun_out/${R}_launches.csv gpurun_out/${R}_launches_summary.txt > /dev/null
python tools/ncu_summary.py full gpurun_out/${R}_full_c5.ncu-rep gpurun_out/${R}_full_c5_summary.txt gpurun_out/${R}_traffic_c5.json > /dev/null
ncu -i gpurun_out/${R}_full_c4.ncu-rep --page source --csv --print-source sass -k "regex:k_gcols" --launch-count 1 \
    > gpurun_out/${R}_sass_k_cols_c4.csv 2>/dev/null
ncu -i gpurun_out/${R}_full_c4.ncu-rep --page source --csv --print-source cuda -k "regex:k_gcols" --launch-count 1 \
    > gpurun_out/${R}_src_k_cols_c4.csv 2>/dev/null
python tools/ncu_summary.py full gpurun_out/${R}_full_c3.ncu-rep gpurun_out/${R}_full_c3_summary.txt gpurun_out/${R}_traffic_c3.json > /dev/null
python tools/ncu_summary.py full gpurun_out/${R}_full_c4.ncu-rep gpurun_out/${R}_full_c4_summary.txt gpurun_out/${R}_traffic_c4.json > /dev/null
for k in k_col_fwd k_col_inv k_row_pmul; do
  ncu -i gpurun_out/${R}_full_c3.ncu-rep --page source --csv --print-source sass -k "regex:$k" --launch-count 1 \
      > gpurun_out/${R}_sass_${k}.csv 2>/dev/null
done
gzip -f gpurun_out/${R}_sass_*.csv
rm -f gpurun_out/${R}_full_c4.ncu-rep gpurun_out/${R}_full_c3.ncu-rep gpurun_out/${R}_full_c5.ncu-rep
ls -la gpurun_out | grep ${R}
du -sh gpurun_out
