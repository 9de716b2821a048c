# multi-GPU iteration: GPU tests (incl. NCCL multirank), bench at N=1 and N=NG via torchrun
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${TAG:-multi}
NG=$(nvidia-smi -L | wc -l)
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1
timeout 300 python bench.py > gpurun_out/${TAG}_bench_n1.json 2> gpurun_out/${TAG}_bench_n1.err
for N in 2 4 8; do
  if [ $N -le $NG ]; then
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 \
      bench.py --gpus $N > gpurun_out/${TAG}_bench_n$N.json 2> gpurun_out/${TAG}_bench_n$N.err
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29512 \
      bench.py --gpus $N --batch 16 > gpurun_out/${TAG}_bench_n${N}_k16.json 2> gpurun_out/${TAG}_bench_n${N}_k16.err
  fi
done
timeout 300 python bench.py --batch 16 --no-cpu-baseline > gpurun_out/${TAG}_bench_n1_k16.json 2> gpurun_out/${TAG}_bench_n1_k16.err
echo done
