# Round evidence in one gpurun session: smoke, GPU suite, bench lines for every
# config (+ variants and the reference arm), the launch list of the timed region
# and ncu --set full captures of the kernels that matter.  Outputs: gpurun_out/ev_*
mkdir -p gpurun_out
timeout 300 python __graft_entry__.py smoke > gpurun_out/ev_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/ev_smoke.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 400 -p no:cacheprovider > gpurun_out/ev_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ev_pytest_gpu.log
python bench.py > gpurun_out/ev_bench_cfg2.json 2> gpurun_out/ev_bench_cfg2.err
for C in cfg1 cfg3 cfg4; do timeout 600 python bench.py --config $C --steps 30 --warmup 3 > gpurun_out/ev_bench_$C.json 2>/dev/null; done
timeout 900 python bench.py --config cfg5 --steps 10 --warmup 3 > gpurun_out/ev_bench_cfg5_1gpu.json 2>/dev/null
timeout 600 python bench.py --lagged 0 --steps 60 --warmup 5 > gpurun_out/ev_bench_cfg2_step_fast.json 2>/dev/null
timeout 600 python bench.py --incremental off --steps 30 --warmup 3 > gpurun_out/ev_bench_cfg2_full_recompute.json 2>/dev/null
timeout 600 python bench.py --config cfg4 --counter dr --steps 20 --warmup 3 > gpurun_out/ev_bench_cfg4_dr.json 2>/dev/null
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/ev_bench_reference.json 2> gpurun_out/ev_bench_reference.err
VATE_PROFILE_REGION=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
   python bench.py --steps 10 --warmup 3 > gpurun_out/ev_launches.csv 2> gpurun_out/ev_ncu_launch_run.log
for K in k_scan_packed16 k_bitmap k_active k_inc_apply k_final_all k_sweep; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" -s 140 -c 1 \
     -o gpurun_out/ev_prof_$K python bench.py --steps 20 --warmup 3 > /dev/null 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_scan_packed16" -s 620 -c 1 \
   -o gpurun_out/ev_prof_cfg4_scan python bench.py --config cfg4 --steps 20 --warmup 3 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_bitmap" -s 620 -c 1 \
   -o gpurun_out/ev_prof_cfg4_bitmap python bench.py --config cfg4 --steps 20 --warmup 3 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_dr_slide" -s 600 -c 1 \
   -o gpurun_out/ev_prof_cfg4_dr_slide python bench.py --config cfg4 --counter dr --steps 5 --warmup 3 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_g0" -s 130 -c 1 \
   -o gpurun_out/ev_prof_k_g0_full python bench.py --steps 20 --warmup 3 --incremental off > /dev/null 2>&1
tail -2 gpurun_out/ev_smoke.log; tail -3 gpurun_out/ev_pytest_gpu.log; ls gpurun_out | head -50
# summaries on the box (gpurun brings back <= 64 MiB): text summaries, then drop
# every report but the cfg 2 scan's
python scripts/ncu_summary.py "gpurun_out/ev_prof_*.ncu-rep" > gpurun_out/ev_ncu_kernels.txt 2>&1
python scripts/launch_summary.py gpurun_out/ev_launches.csv 10 > gpurun_out/ev_launches_summary.txt 2>&1
for f in gpurun_out/ev_prof_*.ncu-rep; do
  case "$f" in *k_scan_packed16*) ;; *) rm -f "$f" ;; esac
done
rm -f gpurun_out/prof_*.ncu-rep
du -sh gpurun_out
