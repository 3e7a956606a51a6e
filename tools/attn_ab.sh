# A/B of the fused attention at the bench shape (mbs 16): correctness tests,
# then the backward under several raster group sizes.
set -x
timeout 600 python -m pytest tests/test_attention_gpu.py -q -x 2>&1 | tail -3
for g in 0 16 32 64 128; do
  WP_BW_GROUP=$g timeout 300 python -c "
import sys; sys.path.insert(0, 'tools'); import attn_bench; attn_bench.main(mbs=16)"
done
