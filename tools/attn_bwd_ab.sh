# Attention A/B at the bench shape (mbs 16, GPT-1.3B heads): kernel tests first
# (bounded), then device time of the fused kernels, causal and not.
timeout 120 python -m pytest tests/test_attention_gpu.py -q -x 2>&1 | tail -2 || exit 1
timeout 120 bash tools/attn_kernels.sh | grep flash; CAUSAL=0 timeout 120 bash tools/attn_kernels.sh | grep flash
