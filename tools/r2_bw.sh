# Attention-backward pass: parity, mbs-16 timings, CTA-0 timeline.
O=gpurun_out
timeout 600 python -m pytest tests/test_attention_gpu.py -q -x -p no:cacheprovider > $O/bw_tests.log 2>&1
tail -3 $O/bw_tests.log
grep -q " passed" $O/bw_tests.log && ! grep -q "failed" $O/bw_tests.log || exit 1
POLYS=3 timeout 300 bash tools/fa_poly_ab.sh > $O/bw_ab.log 2>&1; grep -E "bwd" $O/bw_ab.log
rm -f build/obj/kernels/attention_bwd.cu.o
make EXTRA_NVFLAGS="-DWP_BW_TRACE" -j > $O/bw_trace_build.log 2>&1
for c in 0 1; do CAUSAL=$c timeout 120 python tools/bw_trace_probe.py > $O/bw_trace_c${c}.log 2>&1; done
rm -f build/obj/kernels/attention_bwd.cu.o; make -j > /dev/null 2>&1
