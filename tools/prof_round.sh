# Round profile: default bench line, reference arm, launch list of one step,
# ncu --set full of the dominant kernels.  Outputs under gpurun_out/.
set -x
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1
timeout 600 python bench.py --impl reference > gpurun_out/bench_reference.log 2>&1
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 5200 -c 3737 --csv --log-file gpurun_out/launches.csv $B > gpurun_out/l.log 2>&1
for k in gemm_tc2_kernel flash_fwd_kernel flash_bwd_kernel ln_bwd_dx_rows_cs_k ln_fwd_k; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 40 -c 1 -o gpurun_out/full_$k $B > gpurun_out/full_$k.log 2>&1
done
ls -la gpurun_out
