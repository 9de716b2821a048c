cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; TAG=${TAG:-c5}
for N in ${NS:-12 14 16 18 20}; do
  timeout 900 python bench.py --config cfg5 --n $N --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_n$N.json 2>&1
done
echo done
