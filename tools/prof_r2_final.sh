# Round-2 closing profile (outputs under gpurun_out/, summarised into
# profiles/ on the CPU side with tools/ncu_summary.py and tools/traffic.py).
set -x
O=gpurun_out
timeout 600 python bench.py > $O/f_bench.log 2>&1
timeout 400 python bench.py --impl reference > $O/f_bench_ref.log 2>&1
for m in gpt2-medium-like bert-large-like; do
  timeout 600 python bench.py --model $m --mbs 16 --steps 6 --warmup 3 --no-cpu-baseline --gemm-report > $O/f_b_$m.log 2>&1
done
WP_BENCH_SHARE_GPU=1 timeout 600 python bench.py --gpus 2 --steps 2 --warmup 3 --no-cpu-baseline > $O/f_bench_share2.log 2>&1
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 5200 -c 3737 --csv --log-file $O/f_launches.csv $B > $O/f_l.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_tc2 -s 1 -c 1 -o $O/f_gemm_fc1 python tools/gemm_probe.py 16384 8192 2048 gelu > $O/f_gemm_fc1.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:flash_bwd -s 2 -c 1 -o $O/f_flash_bwd python -c "import sys; sys.path.insert(0, 'tools'); import attn_bench; attn_bench.main(mbs=16, n=1)" > $O/f_flash_bwd.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:flash_fwd -s 2 -c 1 -o $O/f_flash_fwd python -c "import sys; sys.path.insert(0, 'tools'); import attn_bench; attn_bench.main(mbs=16, n=1)" > $O/f_flash_fwd.log 2>&1
for k in ln_fwd_pipe_k ln_bwd_dx_rows_cs_k xent_vec_k; do
  timeout 600 ncu --set full --clock-control none -k regex:$k -s 40 -c 1 -o $O/f_full_$k $B > $O/f_full_$k.log 2>&1
done
ls -la $O | tail -40
