#!/bin/bash
# ablation of the row-GEMM pipeline: 0 full, 1 no epilogue, 2 no B copy, 4 no A split, 7 none
for d in 0 1 2 4 3 7; do
  echo "debug=$d"
  DGNN_UMMA_DEBUG=$d timeout 200 python scripts/kernel_bench.py --only cell_fwd_lstm | tr -d '\n '
  echo
done
