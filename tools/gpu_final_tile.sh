cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; TAG=${TAG:-ft}
timeout 900 python -m pytest tests/test_gpu_tile.py tests/test_gpu_parity.py -q > gpurun_out/${TAG}_pytest.log 2>&1
for N in 14 16 18 20; do
  timeout 600 python bench.py --config cfg5 --n $N --batch 2 --steps 2 --warmup 3 --no-cpu-baseline --no-next2 > gpurun_out/${TAG}_n$N.json 2>&1
done
B="python bench.py --config cfg5 --n 18 --batch 2 --steps 1 --warmup 3 --no-cpu-baseline --no-next2"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"stream_plane" -c 1 -o gpurun_out/${TAG}_prof18 $B > gpurun_out/${TAG}_ncu18.log 2>&1
echo done
