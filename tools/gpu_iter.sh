# Iteration pass on one GPU box: smoke, a chosen pytest selection, A/B bench lines.
#   TAG=... PYSEL="tests/..." BENCH_ARGS="..." VARIANTS="1 2" bash tools/gpu_iter.sh
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; TAG=${TAG:-iter}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/${TAG}_nvsmi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
for V in ${VARIANTS:-0}; do
  timeout 600 python bench.py --steps ${STEPS:-50} --no-cpu-baseline --no-next2 --variant $V ${BENCH_ARGS} > gpurun_out/${TAG}_bench_v$V.json 2> gpurun_out/${TAG}_bench_v$V.err
done
if [ -n "${PYSEL}" ]; then
  timeout 2400 python -m pytest ${PYSEL} -q -rs --durations=15 -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1
fi
if [ -n "${NCU_K}" ]; then
  B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-next2 --variant ${NCU_V:-0} ${BENCH_ARGS}"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${NCU_K}" -c 1 -o gpurun_out/${TAG}_prof $B > gpurun_out/${TAG}_ncu.log 2>&1
fi
echo done
