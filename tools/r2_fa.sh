# Attention-forward pass: parity, poly-share A/B at the bench shapes, then a
# CTA-0 timeline from an instrumented (-DWP_FA_TRACE) rebuild.
O=gpurun_out
timeout 600 python -m pytest tests/test_attention_gpu.py -q -x -p no:cacheprovider > $O/fa_tests.log 2>&1
tail -3 $O/fa_tests.log
grep -q " passed" $O/fa_tests.log && ! grep -q "failed" $O/fa_tests.log || exit 1
timeout 900 bash tools/fa_poly_ab.sh > $O/fa_poly_ab.log 2>&1
grep -E "fwd" $O/fa_poly_ab.log
timeout 900 python -m pytest tests/test_runtime_gpu.py tests/test_parity_bench_dims.py -q -x -p no:cacheprovider > $O/fa_tests2.log 2>&1
tail -3 $O/fa_tests2.log
rm -f build/obj/kernels/attention_fwd.cu.o
make EXTRA_NVFLAGS="-DWP_FA_TRACE" -j > $O/fa_trace_build.log 2>&1
for c in 0 1; do
  timeout 120 python tools/fa_trace_probe.py $c > $O/fa_trace_c${c}.log 2>&1
done
rm -f build/obj/kernels/attention_fwd.cu.o; make -j > /dev/null 2>&1
