# plane2 with c-Z_j folded into the FWHT stage: bitwise parity vs plane_kernel, bench
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; TAG=${TAG:-r2zz}
timeout 900 python -m pytest tests/test_gpu_plane.py tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1
timeout 600 python bench.py --steps 100 --no-cpu-baseline --no-next2 --no-traffic > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
timeout 600 python bench.py --steps 100 --no-cpu-baseline --no-next2 --no-traffic > gpurun_out/${TAG}_bench2.json 2> gpurun_out/${TAG}_bench2.err
echo done
