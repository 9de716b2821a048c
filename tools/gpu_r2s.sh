# after the prefix revert + plane2 pdl_wait move: parity subset, quad stamps, K=1 probe, bench
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; TAG=${TAG:-r2s}
./tools/prefix_timing > gpurun_out/${TAG}_quad_stamps.json 2>&1
timeout 1200 python -m pytest tests/test_gpu_plane.py tests/test_gpu_parity.py tests/test_gpu_solve.py tests/test_gpu_virtual.py tests/test_gpu_p2p_host.py -q -x -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1
timeout 300 python tools/k1_probe.py > gpurun_out/${TAG}_k1_probe.json 2>&1
timeout 600 python bench.py --steps 100 --no-cpu-baseline --no-next2 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo done
