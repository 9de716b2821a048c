# duo prefix: parity (prefix tests), prefix timing, K=1 probe, bench K=16/K=1
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; TAG=${TAG:-r2o}
timeout 900 python -m pytest tests/test_gpu_solve.py tests/test_gpu_plane.py tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1
timeout 300 python tools/prefix_probe.py 1 > gpurun_out/${TAG}_prefix_K1.json 2>&1
timeout 300 python tools/prefix_probe.py 16 > gpurun_out/${TAG}_prefix_K16.json 2>&1
timeout 300 python tools/k1_probe.py > gpurun_out/${TAG}_k1_probe.json 2>&1
timeout 600 python bench.py --steps 100 --no-cpu-baseline --no-next2 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:prefix_duo -s 3 -c 1 -o gpurun_out/${TAG}_prefix python tools/prefix_probe.py 1 > gpurun_out/${TAG}_ncu.log 2>&1
echo done
