# usage: bash scripts/gpu_bf16_unroll.sh (2 GPUs) — bf16-wire FLAT at p = 2: U = 6 (spill-free) vs U = 8, A/B/A via two builds
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 2"
ab() {
  for c in nin alexnet; do
    timeout 300 $TR --master-port 29731 bench.py --gpus 2 --config $c --steps 50 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', '$c', 'bf16_ms', d['baselines_ms_per_step']['flat_bf16_wire_ms'], 'fp32_ms', d['ms_per_step'])"
  done
}
ab U6
sed -i 's/#define BF16_UNROLL(P) ((P) <= 2 ? 6 :/#define BF16_UNROLL(P) ((P) <= 2 ? 8 :/' paper_1511_00175_b200/csrc/coll_flat.cu
python -c "from paper_1511_00175_b200.build import build; build(force=True)" > /dev/null 2>&1
ab U8
sed -i 's/#define BF16_UNROLL(P) ((P) <= 2 ? 8 :/#define BF16_UNROLL(P) ((P) <= 2 ? 6 :/' paper_1511_00175_b200/csrc/coll_flat.cu
python -c "from paper_1511_00175_b200.build import build; build(force=True)" > /dev/null 2>&1
ab U6
