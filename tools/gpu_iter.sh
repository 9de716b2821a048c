# one build->measure iteration on a GPU box: parity tests, bench (default and
# DVQLS_WARPS=12), then one ncu --set full capture of the Hadamard-test kernel.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${TAG:-iter}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
#for W in 8; do DVQLS_WARPS=$W timeout 300 python bench.py --no-cpu-baseline > gpurun_out/${TAG}_bench_w$W.json 2>&1; done
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline"
if [ "${NCU:-1}" = "1" ]; then
timeout 300 $B > gpurun_out/${TAG}_b5.json 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"hadamard" -c 1 -o gpurun_out/${TAG}_prof $B > gpurun_out/${TAG}_ncu.log 2>&1
fi
echo done
