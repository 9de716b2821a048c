# plane2 tail trims: stamps, parity subset, bench
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; TAG=${TAG:-r2z}
./tools/plane2_timing 1 > gpurun_out/${TAG}_stamps_k1.json 2>&1
./tools/plane2_timing 16 > gpurun_out/${TAG}_stamps_k16.json 2>&1
timeout 1200 python -m pytest tests/test_gpu_plane.py tests/test_gpu_parity.py tests/test_gpu_virtual.py tests/test_gpu_p2p_host.py tests/test_gpu_shift.py -q -x -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1
timeout 600 python bench.py --steps 100 --no-cpu-baseline --no-next2 --no-traffic > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo done
