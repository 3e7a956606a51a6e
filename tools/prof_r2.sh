# Round-2 GPU profile pass (outputs under gpurun_out/):
#  - ncu --set full of the FC1-forward GEMM at the bench shape and of the
#    attention backward at the bench shape (profiles/traffic.json inputs)
#  - launch list of one GPT-1.3B step, and of one GPT2-medium / BERT-large step
#  - bench lines of the C2 / C3 presets at P=1 with the per-shape GEMM table
set -x
O=gpurun_out
timeout 300 ncu --set full --clock-control none -k regex:gemm_tc2 -s 2 -c 1 -o $O/r2_gemm_fc1 python tools/gemm_probe.py 16384 8192 2048 gelu > $O/r2_gemm_fc1.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:flash_bwd -s 2 -c 1 -o $O/r2_flash_bwd python -c "import sys; sys.path.insert(0, 'tools'); import attn_bench; attn_bench.main(mbs=16, n=1)" > $O/r2_flash_bwd.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:flash_fwd -s 2 -c 1 -o $O/r2_flash_fwd python -c "import sys; sys.path.insert(0, 'tools'); import attn_bench; attn_bench.main(mbs=16, n=1)" > $O/r2_flash_fwd.log 2>&1
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r2_launches.csv $B > $O/r2_l.log 2>&1
for m in gpt2-medium-like bert-large-like; do
  timeout 600 python bench.py --model $m --mbs 16 --steps 6 --warmup 3 --no-cpu-baseline --gemm-report > $O/r2_b_$m.log 2>&1
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r2_launches_$m.csv python bench.py --model $m --mbs 16 --steps 1 --warmup 1 --no-cpu-baseline > $O/r2_l_$m.log 2>&1
done
ls -la $O | tail -30
