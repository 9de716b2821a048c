# GPU parity of the NEXT-2 / NEXT-3 paths + the default bench line (with the NEXT-2 side measurement).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; TAG=${TAG:-nx}
timeout 1200 python -m pytest tests/test_gpu_pauli.py tests/test_gpu_global.py -x -q > gpurun_out/${TAG}_pytest.log 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo done
