# Full validation pass on one GPU box (round evidence): smoke, all GPU tests, bench (with cpu_baseline and
# the NEXT-2/3/4 side measurements), reference arm, ncu launch list of the bench command, ncu --set full of
# the headline kernel and of the prefix kernel.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; TAG=${TAG:-full}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/${TAG}_nvsmi.txt 2>&1
nproc > gpurun_out/${TAG}_nproc.txt; lscpu | grep "Model name" >> gpurun_out/${TAG}_nproc.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 2400 python -m pytest tests -m gpu -q -rs --durations=25 > gpurun_out/${TAG}_pytest.log 2>&1
timeout 600 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${TAG}_ref.json 2> gpurun_out/${TAG}_ref.err
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-next2 --no-traffic"
timeout 300 $B > gpurun_out/${TAG}_b5.json 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv $B > gpurun_out/${TAG}_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"plane2_kernel" -c 1 -o gpurun_out/${TAG}_prof $B > gpurun_out/${TAG}_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"prefix_quad" -c 1 -o gpurun_out/${TAG}_prefix $B > gpurun_out/${TAG}_ncu_prefix.log 2>&1
echo done
