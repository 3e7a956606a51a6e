# Attention backward (16 softmax warps) + pair-GEMM epilogue prefetch: parity,
# timings, trace; GEMM epilogue-mode A/B.
O=gpurun_out
timeout 600 python -m pytest tests/test_attention_gpu.py tests/test_gemm_gpu.py -q -x -p no:cacheprovider > $O/bw2_tests.log 2>&1
tail -3 $O/bw2_tests.log
grep -q " passed" $O/bw2_tests.log && ! grep -q "failed" $O/bw2_tests.log || exit 1
POLYS=3 timeout 300 bash tools/fa_poly_ab.sh > $O/bw2_ab.log 2>&1; grep -E "bwd" $O/bw2_ab.log
timeout 300 python tools/gemm_epi_bench.py > $O/epi_pre.log 2>&1; cat $O/epi_pre.log
WP_GEMM_NO_EPI_PREFETCH=1 timeout 300 python tools/gemm_epi_bench.py > $O/epi_nopre.log 2>&1; cat $O/epi_nopre.log
rm -f build/obj/kernels/attention_bwd.cu.o
make EXTRA_NVFLAGS="-DWP_BW_TRACE" -j > $O/bw_trace_build.log 2>&1
for c in 0 1; do CAUSAL=$c timeout 120 python tools/bw_trace_probe.py > $O/bw_trace_c${c}.log 2>&1; done
rm -f build/obj/kernels/attention_bwd.cu.o; make -j > /dev/null 2>&1
