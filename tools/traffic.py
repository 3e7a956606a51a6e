"""profiles/traffic.json entries from `ncu --set full` captures: DRAM bytes
per launch (dram__bytes_read.sum + dram__bytes_write.sum) next to the
launch's algorithmic bytes, keyed by what bench.py looks up:

  gemm_fc1   FC1 forward (GELU epilogue) at the bench shape, M = mbs*seq,
             N = ffn, K = hidden: A + B + C + pre-activation aux, bf16
  flash_bwd  fused attention backward at the bench shape: QKV, dO in,
             dQKV out (bf16), lse and Delta (fp32), the fp32 dQ accumulator
             written once

    python tools/traffic.py gemm_fc1 <rep> M N K
    python tools/traffic.py flash_bwd <rep> mbs heads seq d causal
"""
import csv
import io
import json
import os
import subprocess
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def dram_bytes(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units, v = rows[0], rows[1], rows[2]
    get = lambda k: float(v[h.index(k)].replace(",", "")) * SCALE.get(units[h.index(k)], 1)
    t = float(v[h.index("gpu__time_duration.sum")].replace(",", ""))
    t_us = t / 1e3 if units[h.index("gpu__time_duration.sum")] in ("nsecond", "ns") else t
    return get("dram__bytes_read.sum"), get("dram__bytes_write.sum"), t_us


def main():
    key, rep = sys.argv[1], sys.argv[2]
    dims = [int(x) for x in sys.argv[3:]]
    if key == "gemm_fc1":
        M, N, K = dims
        alg = 2 * (M * K + N * K + 2 * M * N)
        kernel = "gemm_tc2_kernel (FC1 forward, bias + GELU epilogue, pre-activation stored)"
    elif key == "flash_bwd":
        mbs, heads, seq, d, causal = dims
        T, h = mbs * seq, heads * d
        alg = 2 * (3 * T * h + T * h + 3 * T * h) + 8 * mbs * heads * seq + 4 * T * h
        kernel = "flash_bwd_kernel<%d> (causal=%d)" % (d, causal)
    else:
        raise SystemExit("unknown key " + key)
    rd, wr, us = dram_bytes(rep)
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "traffic.json")
    try:
        with open(path) as f:
            allj = json.load(f)
    except (OSError, ValueError):
        allj = {}
    allj[key] = {"kernel": kernel, "shape": dims, "bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
                 "algorithmic_bytes": alg, "ratio": (rd + wr) / alg, "duration_us": us,
                 "source": os.path.basename(rep)}
    with open(path, "w") as f:
        json.dump(allj, f, indent=1)
    print(json.dumps(allj[key], indent=1))


if __name__ == "__main__":
    main()
