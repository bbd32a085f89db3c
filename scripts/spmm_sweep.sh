#!/bin/bash
# slice-count sweep for the pull SpMMs at C3 shapes
for s in 1 2 4 8 16; do
  echo "slices=$s"
  DGNN_SPMM_SLICES=$s timeout 200 python scripts/kernel_bench.py --only agg_scratch64,agg_backward64,agg_scratch128 | tr -d '\n '
  echo
done
