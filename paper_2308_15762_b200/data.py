"""Synthetic token batches: t[i] = splitmix64(seed ^ i) mod V.

GPT-like: labels are the inputs shifted by one (each sequence draws seq+1
tokens).  BERT-like: labels on every position, drawn from an independent
stream (MLM-style targets).
"""
import numpy as np

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(x):
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = x + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def synthetic_batch(microbatches, micro_batch_size, seq, vocab, causal=True, seed=0x5EED, step=0):
    """(tokens, labels) int32 [B, mbs, seq]."""
    n_seq = microbatches * micro_batch_size
    base = np.uint64(seed) ^ (np.uint64(step) << np.uint64(40))
    if causal:
        idx = np.arange(n_seq * (seq + 1), dtype=np.uint64)
        stream = (splitmix64(base ^ idx) % np.uint64(vocab)).astype(np.int32).reshape(n_seq, seq + 1)
        tokens, labels = stream[:, :seq], stream[:, 1:]
    else:
        idx = np.arange(n_seq * seq, dtype=np.uint64)
        tokens = (splitmix64(base ^ idx) % np.uint64(vocab)).astype(np.int32).reshape(n_seq, seq)
        labels = (splitmix64(base ^ (idx + np.uint64(1 << 39))) % np.uint64(vocab)).astype(np.int32)
        labels = labels.reshape(n_seq, seq)
    shape = (microbatches, micro_batch_size, seq)
    return np.ascontiguousarray(tokens.reshape(shape)), np.ascontiguousarray(labels.reshape(shape))
