# usage: bash scripts/gpu_host_stages.sh N  — e2e of the multi-GPU host entry point vs pipeline stages
# (profiles/r01_host_stages_n*.jsonl)
N=${1:-2}
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node $N"
for S in 1 2 4 8; do
  FC_HOST_STAGES=$S timeout 600 $TR --master-port $((29700 + S)) bench.py --gpus $N --steps 50 --warmup 5 --no-baselines \
    2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print(json.dumps({'n_gpus': $N, 'stages': $S, 'e2e_gbs': d['e2e']['value'], 'e2e_ms': d['e2e'].get('ms_per_step'), 'device_ms': d['ms_per_step'], 'bitexact': d['parity']['bitexact_sampled']}))"
done
