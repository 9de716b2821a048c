# n = 11, 12 two-exchange kernel: tile-path parity, cfg5 n = 12 bench (default vs DVQLS_ONCHIP=0), ncu
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; TAG=${TAG:-oc}
timeout 1200 python -m pytest tests/test_gpu_tile.py tests/test_multirank.py -q -x > gpurun_out/${TAG}_pytest.log 2>&1
timeout 600 python bench.py --config cfg5 --n 12 --batch 2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_n12.json 2>&1
DVQLS_ONCHIP=0 timeout 600 python bench.py --config cfg5 --n 12 --batch 2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_n12_tile.json 2>&1
B="python bench.py --config cfg5 --n 12 --batch 2 --steps 1 --warmup 3 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"onchip_plane" -c 1 -o gpurun_out/${TAG}_prof $B > gpurun_out/${TAG}_ncu.log 2>&1
echo done
