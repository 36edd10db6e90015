# Round-2 evidence run: sanitizers on small problems, ncu --set full captures of the
# shipped top kernels, the bench launch list. Outputs under gpurun_out/ (summarised
# into profiles/r02_* by tools/summarize_evidence.py).
mkdir -p gpurun_out
for tool in racecheck synccheck memcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_probe.py \
    > gpurun_out/sanitizer_$tool.log 2>&1
  echo "sanitizer $tool rc=$?" >> gpurun_out/sanitizer_rc.log
done
# the bench's launch list (C4; serialised, cold-cache: shares, not absolutes)
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -c 1300 --csv --log-file gpurun_out/r02b_c4_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
  --no-c5 --no-per-level --e2e-steps 1 > gpurun_out/ncu_launch.log 2>&1
# full captures (one launch each)
bash tools/ncu_capture.sh r02b_walk_norm k_ss_walk 0 python tools/profile_cycle.py --cycles 1
bash tools/ncu_capture.sh r02b_walk_arr k_ss_walk 29 python tools/profile_cycle.py --cycles 1
bash tools/ncu_capture.sh r02b_scan_chain k_ss_scan_chain 0 python tools/profile_cycle.py --cycles 1
bash tools/ncu_capture.sh r02b_resid4 k_resid4 0 python tools/profile_cycle.py --cycles 1
bash tools/ncu_capture.sh r02b_smooth4_correct k_smooth4 0 python tools/smoother_probe.py --levels 13 --alphas 1 --steps 2 --variants 1 --reps 1
bash tools/ncu_capture.sh r02b_smooth4_pe k_smooth4 0 python tools/smoother_probe.py --levels 13 --alphas 1 --steps 2 --variants 0 --reps 1
bash tools/ncu_capture.sh r02b_smooth4_c5_m3 k_smooth4 0 python tools/smoother_probe.py --levels 14 --alphas 1e-2 --steps 3 --variants 1 --reps 1
bash tools/ncu_capture.sh r02b_omega4 k_omega4 0 python tools/profile_cycle.py --cycles 1

ls -la gpurun_out
bash tools/ncu_capture.sh r02b_gs_wave k_gs_wave 0 python tools/gs_step.py 10 1e-2

rm -f gpurun_out/*.sass.csv; ls gpurun_out | head -80
