"""profiles/gemm_traffic.json from an `ncu --set full` capture of the CTA-pair
GEMM on the step's most expensive shape (FC1 forward, GELU epilogue:
M = mbs*seq = 8192 tokens, N = ffn 8192, K = hidden 2048): DRAM bytes per
launch next to the algorithmic bytes (A + B + C + aux, bf16).

    ncu --set full -k regex:gemm_tc2 -c 1 -o gpurun_out/gemm_fc1 \
        python tools/gemm_probe.py 8192 8192 2048 gelu
    python tools/gemm_traffic.py gpurun_out/gemm_fc1.ncu-rep
"""
import csv
import io
import json
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, v = rows[0], rows[-1]
m = dict(zip(h, v))
rd = float(m["dram__bytes_read.sum"])
wr = float(m["dram__bytes_write.sum"])
unit_rd = rows[1][h.index("dram__bytes_read.sum")]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
rd *= scale.get(unit_rd, 1)
wr *= scale.get(rows[1][h.index("dram__bytes_write.sum")], 1)
M, N, K = 8192, 8192, 2048
alg = 2 * (M * K + N * K + 2 * M * N)  # A, B, C and the pre-activation aux output
res = {"kernel": "gemm_tc2_kernel (FC1 forward, GELU epilogue)", "shape": [M, N, K],
       "bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr, "algorithmic_bytes": alg,
       "ratio": (rd + wr) / alg, "duration_us": float(m["gpu__time_duration.sum"]) / 1e3
       if rows[1][h.index("gpu__time_duration.sum")] == "nsecond" else float(m["gpu__time_duration.sum"]),
       "source": rep}
print(json.dumps(res, indent=1))
with open("profiles/gemm_traffic.json", "w") as f:
    json.dump(res, f, indent=1)
