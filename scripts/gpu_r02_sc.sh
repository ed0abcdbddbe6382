# usage: bash scripts/gpu_r02_sc.sh  (under gpurun --gpus 2): fence.sc.sys build -- parity, bench N=2 NiN/GoogLeNet x2,
# one-clock breakdown; the load-variant exit decomposition (gap_bench)
O=gpurun_out/r02_sc; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 2"
FC_MP_TIMEOUT=5 FC_MP_STRESS=300 timeout 900 $TR --master-port 29621 tests/mp_worker.py > $O/mp.log 2>&1
echo "parity rc=$? ok=$(grep -o 'MP_OK' $O/mp.log | wc -l)" >> $O/summary.txt
for rep in 1 2; do for c in nin googlenet; do
  timeout 600 $TR --master-port 29622 bench.py --gpus 2 --config $c --steps 200 --warmup 20 --no-baselines --no-cpu-baseline > $O/b.json 2>/dev/null
  echo "rep$rep $c $(python -c "import json;d=json.load(open('$O/b.json'));print(d['ms_per_step'], d['parity']['bitexact_sampled'])")" >> $O/summary.txt
done; done
timeout 300 $TR --master-port 29623 scripts/gap_coll.py --size 7600000 2>/dev/null | grep '"fused"' >> $O/summary.txt
timeout 300 ./scripts/gap_bench > $O/gap_bench.txt 2>&1
echo done
