# usage: bash scripts/gpu_sgd_db.sh — 1-GPU SGD: plain vs register double-buffered (--sgd-unroll), all configs, A/B/A/B
for rep in 1 2; do
for c in nin googlenet alexnet vgg19; do
  for u in 4 -2 -4 -1; do
    timeout 300 python bench.py --config $c --steps 100 --warmup 5 --no-baselines --no-cpu-baseline --sgd-unroll=$u 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print(json.dumps({'config': '$c', 'sgd_unroll': $u, 'rep': $rep, 'ms': d['ms_per_step'], 'frac': d['roofline']['frac'], 'bitexact': d['parity']['bitexact_sampled']}))"
  done
done
done
