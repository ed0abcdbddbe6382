#!/bin/bash
# torchrun --no-python entry: rank 0 runs under ncu (single-pass NVLink byte metrics, one launch), every other
# rank runs plainly -- so the profiled cross-GPU kernel has live peers (kernel replay would need them twice).
#   torchrun --nproc-per-node 2 --no-python scripts/ncu_rank0.sh OUT.csv scripts/real_flat_run.py nin
OUT=$1; shift
if [ "${LOCAL_RANK:-0}" = "0" ]; then
  exec ncu --metrics nvlrx__bytes.sum,nvltx__bytes.sum --cache-control none --clock-control none \
    -k regex:flat_kernel -s 3 -c 1 --csv --log-file "$OUT" python "$@"
else
  exec python "$@"
fi
