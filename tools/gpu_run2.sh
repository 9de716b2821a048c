cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
timeout 300 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline"
timeout 300 $B > gpurun_out/b5.json 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"hadamard|prefix" -c 2 -o gpurun_out/prof_r1 $B > gpurun_out/ncu_full.log 2>&1
echo done
