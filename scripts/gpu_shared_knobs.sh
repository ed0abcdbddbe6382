# usage: bash scripts/gpu_shared_knobs.sh — 8 ranks on 4 GPUs (2 per GPU) under every forced kernel build /
# exit protocol / mapping: co-located ranks time-slice, so every protocol sees adversarial CTA timing
i=0
for K in "" "FC_EXIT=cta" "FC_TREE_CTAS_PER_SM=2 FC_FLAT_UNROLL=1 FC_FLAT_CTAS_PER_SM=2" "FC_FLAT_MAP=stride" "FC_HOST_STAGES=3 FC_TREE_CTAS_PER_SM=1" "FC_LAUNCH=coop"; do
  i=$((i+1))
  env $K FC_MP_GPUS=4 FC_MP_SIZES=5,16391,300007 FC_MP_STRESS=100 FC_MP_TIMEOUT=30 FC_MP_TIMEOUT_TEST=0 timeout 600 \
    python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 8 --master-port $((29720 + i)) tests/mp_worker.py > gpurun_out/shk_$i.log 2>&1
  echo "[$K] rc=$? ok=$(grep -o 'MP_OK [0-9]' gpurun_out/shk_$i.log | wc -l)"; grep -h FAILS gpurun_out/shk_$i.log | cut -c1-200 | head -3
done
