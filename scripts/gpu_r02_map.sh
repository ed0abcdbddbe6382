# usage: bash scripts/gpu_r02_map.sh N   (under gpurun --gpus N): FLAT work mapping balanced vs dyn
# (A/B/A/B, one-clock breakdown + bench at NiN), parity of dyn first; exit protocol decomposition (N=2)
N=${1:-2}
mkdir -p gpurun_out
O=gpurun_out/r02_map_n$N.txt
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
if [ "$N" = 2 ]; then timeout 300 ./scripts/gap_bench > gpurun_out/r02_gap_bench.txt 2>&1; fi
FC_FLAT_MAP=dyn FC_MP_TIMEOUT=5 FC_MP_TIMEOUT_TEST=0 FC_MP_STRESS=400 timeout 900 $TR --master-port 29551 tests/mp_worker.py > gpurun_out/r02_map_mp_dyn_n$N.log 2>&1
echo "dyn parity rc=$? ok=$(grep -o 'MP_OK' gpurun_out/r02_map_mp_dyn_n$N.log | wc -l)" >> $O
for rep in 1 2; do for M in balanced dyn; do
  FC_FLAT_MAP=$M timeout 300 $TR --master-port 29552 scripts/gap_coll.py --size 7600000 --dump 2>/dev/null | grep '"fused"' | sed "s/^/$M rep$rep /" >> $O
done; done
for rep in 1 2; do for M in balanced dyn; do
  FC_FLAT_MAP=$M timeout 600 $TR --master-port 29553 bench.py --gpus $N --steps 200 --warmup 20 --no-baselines --no-cpu-baseline > gpurun_out/r02_map_bench_${M}_n$N.json 2>/dev/null
  echo "$M rep$rep bench $(python -c "import json;d=json.load(open('gpurun_out/r02_map_bench_${M}_n$N.json'));print(d['ms_per_step'], d['parity']['bitexact_sampled'], d['parity'].get('executors'))")" >> $O
done; done
for M in balanced dyn; do for c in googlenet alexnet; do
  FC_FLAT_MAP=$M timeout 600 $TR --master-port 29554 bench.py --gpus $N --config $c --steps 50 --warmup 5 --no-baselines --no-cpu-baseline > gpurun_out/r02_map_bench_${M}_${c}_n$N.json 2>/dev/null
  echo "$M $c bench $(python -c "import json;d=json.load(open('gpurun_out/r02_map_bench_${M}_${c}_n$N.json'));print(d['ms_per_step'], d['parity']['bitexact_sampled'])")" >> $O
done; done
echo done
