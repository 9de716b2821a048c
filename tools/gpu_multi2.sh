cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; TAG=${TAG:-mm}
NG=$(nvidia-smi -L | wc -l)
timeout 900 python -m pytest tests/test_multirank.py tests/test_gpu_parity.py -x -q > gpurun_out/${TAG}_pytest.log 2>&1
for N in 2 4 8; do
  if [ $N -le $NG ]; then
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 \
      bench.py --gpus $N > gpurun_out/${TAG}_bench_n$N.json 2> gpurun_out/${TAG}_bench_n$N.err
    DVQLS_ALLREDUCE=nccl timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29512 \
      bench.py --gpus $N > gpurun_out/${TAG}_bench_n${N}_nccl.json 2> gpurun_out/${TAG}_bench_n${N}_nccl.err
  fi
done
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/${TAG}_bench_n1.json 2> gpurun_out/${TAG}_bench_n1.err
echo done
