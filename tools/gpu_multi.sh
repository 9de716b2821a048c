# Multi-GPU pass on one box (gpurun --gpus N): NCCL/P2P parity under torchrun, strong scaling of cfg3
# (K = 16 headline and K = 1 in every line) at 1..N GPUs with the fused NVLink reduction and with the
# NCCL fallback, cfg4 at 1 and N GPUs, and the 1-GPU weak-scaling reference (rank 0's block of an
# N-way split as a virtual rank).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; TAG=${TAG:-m4}
NG=$(nvidia-smi -L | wc -l); echo "gpus=$NG" > gpurun_out/${TAG}_info.txt
nvidia-smi topo -m >> gpurun_out/${TAG}_info.txt 2>&1
timeout 1200 python -m pytest tests/test_multirank.py -x -q > gpurun_out/${TAG}_pytest.log 2>&1
P=29600
for N in 1 2 4 8; do
  if [ $N -le $NG ]; then
    P=$((P+1))
    if [ $N -eq 1 ]; then
      timeout 600 python bench.py --no-cpu-baseline --no-next2 > gpurun_out/${TAG}_cfg3_n1.json 2> gpurun_out/${TAG}_cfg3_n1.err
    else
      timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $P \
        bench.py --gpus $N --no-next2 > gpurun_out/${TAG}_cfg3_n$N.json 2> gpurun_out/${TAG}_cfg3_n$N.err
      P=$((P+1))
      timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
        --master-port $P bench.py --gpus $N --no-next2 --allreduce nccl > gpurun_out/${TAG}_cfg3_n${N}_nccl.json 2> gpurun_out/${TAG}_cfg3_n${N}_nccl.err
    fi
  fi
done
timeout 600 python bench.py --config cfg4 --no-cpu-baseline --no-next2 --steps 50 > gpurun_out/${TAG}_cfg4_n1.json 2> gpurun_out/${TAG}_cfg4_n1.err
timeout 600 python bench.py --config cfg4 --no-cpu-baseline --no-next2 --steps 50 --slice $NG > gpurun_out/${TAG}_cfg4_slice$NG.json 2> gpurun_out/${TAG}_cfg4_slice$NG.err
P=$((P+1))
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port $P \
  bench.py --gpus $NG --config cfg4 --no-next2 --steps 50 > gpurun_out/${TAG}_cfg4_n$NG.json 2> gpurun_out/${TAG}_cfg4_n$NG.err
P=$((P+1))
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port $P \
  bench.py --impl reference --gpus $NG --steps 3 --warmup 1 > gpurun_out/${TAG}_ref_n$NG.json 2> gpurun_out/${TAG}_ref_n$NG.err
echo done
