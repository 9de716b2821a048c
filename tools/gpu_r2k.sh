cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; TAG=r2k
timeout 1200 python -m pytest tests/test_gpu_tile.py tests/test_gpu_virtual.py -q -x > gpurun_out/${TAG}_pytest.log 2>&1
for N in 14 16 18 20; do for V in 0 4 3; do
  timeout 900 python bench.py --config cfg5 --n $N --batch 2 --steps 2 --warmup 3 --no-cpu-baseline --variant $V > gpurun_out/${TAG}_c5_n${N}_v$V.json 2>&1
done; done
echo done
