# usage: bash scripts/gpu_r02_soak.sh  (under gpurun --gpus 4): soak of the final build -- 5000 random back-to-back
# collectives (op, executor, size; no host sync) on a real 4-GPU world, 2000 on an 8-rank world sharing the 4 GPUs,
# 1500 on a 2-rank world sharing ONE GPU
O=gpurun_out/r02_soak; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
FC_MP_TIMEOUT=10 FC_MP_STRESS=5000 timeout 1500 $TR --nproc-per-node 4 --master-port 29671 tests/mp_worker.py > $O/soak_4gpu.log 2>&1
echo "4 ranks / 4 GPUs, 5000 calls: rc=$? ok=$(grep -o 'MP_OK' $O/soak_4gpu.log | wc -l)" >> $O/summary.txt
FC_MP_GPUS=4 FC_MP_SIZES=5,16391,300007 FC_MP_TIMEOUT=30 FC_MP_TIMEOUT_TEST=0 FC_MP_STRESS=2000 timeout 1500 $TR --nproc-per-node 8 --master-port 29672 tests/mp_worker.py > $O/soak_8on4.log 2>&1
echo "8 ranks / 4 GPUs, 2000 calls: rc=$? ok=$(grep -o 'MP_OK' $O/soak_8on4.log | wc -l)" >> $O/summary.txt
FC_MP_GPUS=1 FC_MP_SIZES=5,16391,300007 FC_MP_TIMEOUT=30 FC_MP_TIMEOUT_TEST=0 FC_MP_STRESS=1500 CUDA_VISIBLE_DEVICES=0 timeout 1500 $TR --nproc-per-node 2 --master-port 29673 tests/mp_worker.py > $O/soak_2on1.log 2>&1
echo "2 ranks / 1 GPU, 1500 calls: rc=$? ok=$(grep -o 'MP_OK' $O/soak_2on1.log | wc -l)" >> $O/summary.txt
echo done
