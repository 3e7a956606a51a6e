# compute-sanitizer over small GPU tests (the mbarrier / TMEM / TMA kernels:
# tcgen05 GEMMs, fused attention, LayerNorm / xent / AdamW, one runtime step,
# the IPC wait kernels).  Summaries to gpurun_out/r2_sanitize_<tool>.log.
O=gpurun_out
T="tests/test_attention_gpu.py tests/test_gemm_gpu.py::test_tc_epilogues tests/test_gemm_gpu.py::test_tc_pair_tma_epilogue_ragged tests/test_ops_gpu.py tests/test_runtime_gpu.py::test_bf16_parity tests/test_runtime_gpu.py::test_fp32_tiny_hanayo_p4_w2_b8"
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --target-processes all --print-limit 20 \
    python -m pytest $T -q -x -p no:cacheprovider > $O/r2_sanitize_$tool.log 2>&1
  echo "== $tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed" $O/r2_sanitize_$tool.log | tail -4
done
