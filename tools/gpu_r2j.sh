cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; TAG=r2j
timeout 900 python -m pytest tests/test_gpu_tile.py -q -k "onchip or full_parity" > gpurun_out/${TAG}_pytest.log 2>&1
for N in 11 12; do for V in 0 4; do
  timeout 600 python bench.py --config cfg5 --n $N --batch 2 --steps 10 --warmup 3 --no-cpu-baseline --variant $V > gpurun_out/${TAG}_c5_n${N}_v$V.json 2>&1
done; done
for N in 14 16; do
  timeout 900 python bench.py --config cfg5amp --n $N --batch 2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_c5amp_n$N.json 2>&1
done
echo done
