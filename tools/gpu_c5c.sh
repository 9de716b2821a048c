cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; TAG=c5c
timeout 600 python -m pytest tests/test_gpu_tile.py -x -q > gpurun_out/${TAG}_pytest.log 2>&1
NS="12 14 16 18 20" NCU=0 TAG=$TAG bash tools/gpu_cfg5.sh
for G in 74 148; do DVQLS_STREAM_GRID=$G timeout 600 python bench.py --config cfg5 --n 16 --batch 2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_n16_g$G.json 2>&1; done
DVQLS_STREAM_GRID=148 timeout 600 python bench.py --config cfg5 --n 14 --batch 2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_n14_g148.json 2>&1
B="python bench.py --config cfg5 --n 18 --batch 2 --steps 1 --warmup 3 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"stream_hadamard" -c 1 -o gpurun_out/${TAG}_prof18 $B > gpurun_out/${TAG}_ncu18.log 2>&1
B="python bench.py --config cfg5 --n 12 --batch 2 --steps 1 --warmup 3 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"stream_hadamard" -c 1 -o gpurun_out/${TAG}_prof12 $B > gpurun_out/${TAG}_ncu12.log 2>&1
