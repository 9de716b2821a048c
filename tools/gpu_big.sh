cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; TAG=${TAG:-big}
free -g > gpurun_out/${TAG}_mem.txt
timeout 1500 python tools/big_parity.py > gpurun_out/${TAG}_parity.log 2>&1
for N in 22 24; do
  timeout 1500 python bench.py --config cfg5 --n $N --batch 2 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/${TAG}_n$N.json 2>&1
done
echo done
