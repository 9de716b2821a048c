# Python binding: cached per-call buffers and plain-address argtypes for dvqls_cost / dvqls_cost_batch
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; TAG=${TAG:-r2py}
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1
timeout 600 python bench.py --steps 100 --no-cpu-baseline --no-next2 --no-traffic > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo done
