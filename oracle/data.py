"""Synthetic input stream of SURVEY.md 8(d) -- TEST / BASELINE INFRASTRUCTURE.

t[i] = splitmix64(seed ^ i) mod V over (microbatch, sample, position); GPT
labels are the stream shifted by one (each sequence draws seq+1 tokens);
BERT-like labels come from an independent stream (offset 2^39).  A
restatement of the input spec (not an import of the product's
paper_2308_15762_b200/data.py), so bench.py's reference arm and the oracle
tests never load the product library; tests/test_oracle.py checks both
produce identical batches.
"""
import numpy as np


def _splitmix64(x):
    z = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = z + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def synthetic_batch(microbatches, micro_batch_size, seq, vocab, causal=True, seed=0x5EED, step=0):
    """(tokens, labels) int32 [B, mbs, seq]."""
    rows = microbatches * micro_batch_size
    key = np.uint64(seed) ^ (np.uint64(step) << np.uint64(40))
    width = seq + 1 if causal else seq
    i = np.arange(rows * width, dtype=np.uint64)
    draw = (_splitmix64(key ^ i) % np.uint64(vocab)).astype(np.int32).reshape(rows, width)
    if causal:
        tokens, labels = draw[:, :-1], draw[:, 1:]
    else:
        tokens = draw
        labels = (_splitmix64(key ^ (i + np.uint64(1 << 39))) % np.uint64(vocab)).astype(np.int32)
        labels = labels.reshape(rows, width)
    shape = (microbatches, micro_batch_size, seq)
    return np.ascontiguousarray(tokens.reshape(shape)), np.ascontiguousarray(labels.reshape(shape))
