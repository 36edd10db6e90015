# Round-2 closing evidence: GS wavefront capture, the finest-level omega-term kernel, the C2 launch
# list and the default bench line (ours + reference arm). Outputs under gpurun_out/.
mkdir -p gpurun_out
bash tools/ncu_capture.sh r02b_gs_wave k_gs_wave 0 python tools/gs_step.py 10 1e-2
bash tools/ncu_capture.sh r02b_omega4_l13 k_omega4 20 python tools/profile_cycle.py --cycles 1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv \
  --log-file gpurun_out/r02b_c2_launches.csv python tools/profile_c2.py 1 > gpurun_out/ncu_c2.log 2>&1
rm -f gpurun_out/*.sass.csv
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench_final.json 2> gpurun_out/bench_final.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02_bench_reference.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
python tools/c2_timing.py > gpurun_out/c2_timing.log 2>&1
python tools/cycle_profile.py --workload C4 > gpurun_out/cycprof_c4.log 2>&1
python tools/cycle_profile.py --workload C5 --skips 0,4,9 > gpurun_out/cycprof_c5.log 2>&1
