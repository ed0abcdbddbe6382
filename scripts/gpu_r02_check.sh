# usage: bash scripts/gpu_r02_check.sh  (under gpurun --gpus 4): parity of the exact final build on real worlds
# (p = 4, 2, 3; 500-call stress), the multi-GPU and DP-training tests, and the rank-0-only ncu NVLink-bytes attempt
O=gpurun_out/r02_check; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for N in 4 3 2; do
  FC_MP_TIMEOUT=5 FC_MP_STRESS=500 timeout 900 $TR --nproc-per-node $N --master-port 2965$N tests/mp_worker.py > $O/mp_n$N.log 2>&1
  echo "N=$N parity rc=$? ok=$(grep -o 'MP_OK' $O/mp_n$N.log | wc -l)" >> $O/summary.txt
  grep "NCCL_TOL" $O/mp_n$N.log | head -3 >> $O/summary.txt
done
timeout 1500 python -m pytest tests/test_multi_gpu.py tests/test_dp_train.py -q -m gpu > $O/pytest_mgpu.log 2>&1; echo "pytest exit $?" >> $O/summary.txt
tail -2 $O/pytest_mgpu.log >> $O/summary.txt
CUDA_VISIBLE_DEVICES=0,1 bash scripts/gpu_r02_nvl2.sh
echo done
