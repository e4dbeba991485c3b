set -u
for c in c1 c2 c4 c5; do
  timeout 600 python bench.py --config $c > gpurun_out/r12_bench_$c.json 2> gpurun_out/r12_bench_$c.err; echo "$c rc=$?"
done
python tools/prof_run.py c5 > gpurun_out/r12_plain_c5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:k_gcols|k_gpmul|k_cols|k_rows|k_carry" -s 7 -c 7 \
    -o gpurun_out/r12_full_c5 python tools/prof_run.py c5 > gpurun_out/r12_ncu_full_c5.log 2>&1
echo c5prof rc=$?
python tools/ncu_summary.py full gpurun_out/r12_full_c5.ncu-rep gpurun_out/r12_full_c5_summary.txt gpurun_out/r12_traffic_c5.json > /dev/null
rm -f gpurun_out/r12_full_c5.ncu-rep
