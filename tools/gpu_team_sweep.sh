cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; TAG=${TAG:-ts}
timeout 900 python -m pytest tests/test_gpu_decomp.py -x -q > gpurun_out/${TAG}_decomp.log 2>&1
for N in 16 18; do
  for MB in 20 40; do
    DVQLS_TEAM_L2_MB=$MB timeout 600 python bench.py --config cfg5 --n $N --batch 2 --steps 2 --warmup 3 --no-cpu-baseline --no-next2 > gpurun_out/${TAG}_n${N}_mb$MB.json 2>&1
  done
  DVQLS_NO_TEAM=1 timeout 600 python bench.py --config cfg5 --n $N --batch 2 --steps 2 --warmup 3 --no-cpu-baseline --no-next2 > gpurun_out/${TAG}_n${N}_noteam.json 2>&1
done
echo done
