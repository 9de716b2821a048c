cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; TAG=r2i
timeout 900 python -m pytest tests/test_gpu_decomp.py -q > gpurun_out/${TAG}_pytest.log 2>&1
timeout 600 python bench.py --steps 20 --no-cpu-baseline > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
for N in 16 18 20; do for V in 0 3; do
  timeout 900 python bench.py --config cfg5 --n $N --batch 2 --steps 2 --warmup 3 --no-cpu-baseline --variant $V > gpurun_out/${TAG}_c5_n${N}_v$V.json 2>&1
done; done
echo done
