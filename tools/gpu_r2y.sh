# zero-copy host-buffer cost calls: parity (every test using dvqls_cost / cost_batch), bench e2e
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; TAG=${TAG:-r2y}
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1
timeout 600 python bench.py --steps 100 --no-cpu-baseline --no-next2 --no-traffic > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
timeout 900 python bench.py --config cfg5 --n 16 --batch 2 --steps 3 --warmup 3 --no-cpu-baseline --no-next2 --no-traffic > gpurun_out/${TAG}_c5n16.json 2>&1
echo done
