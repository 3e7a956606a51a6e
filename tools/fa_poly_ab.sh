# A/B of the attention forward's polynomial-exp2 share (WP_FA_POLY = pairs of
# every 8 on the FMA pipe): mbs-16 timings per setting, D = 128 (GPT-1.3B)
# and D = 64 (GPT2-medium causal, BERT-large seq 512 bidirectional).
for n in ${POLYS:-0 2 3 4 3}; do
  echo "== WP_FA_POLY=$n"
  WP_FA_POLY=$n timeout 300 python -c "
import sys; sys.path.insert(0, 'tools'); import attn_bench as a
a.main(mbs=16); a.main(mbs=16, causal=0); a.main(mbs=16, d=64); a.main(mbs=16, d=64, seq=512, causal=0)"
done
