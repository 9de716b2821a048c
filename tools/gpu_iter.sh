cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; TAG=r2a
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/${TAG}_nvsmi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 600 python bench.py --steps 50 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
timeout 2400 python -m pytest tests -m gpu -q -rs --durations=30 -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1
echo done
