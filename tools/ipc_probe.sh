# Quick multi-process IPC transport probe on one GPU (2 ranks on cuda:0).
set -x
export WP_BENCH_SHARE_GPU=1
timeout 240 python -m pytest tests/test_multiproc_gpu.py -x -q -k "2-4-2" > gpurun_out/mp1.log 2>&1; tail -40 gpurun_out/mp1.log
