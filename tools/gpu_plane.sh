# plane-kernel iteration: n=10 parity, bench (plane default vs DVQLS_PLANE=0, warp variants), ncu of the plane kernel
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; TAG=${TAG:-plane}
timeout 900 python -m pytest tests/test_gpu_plane.py tests/test_gpu_parity.py tests/test_gpu_decomp.py -q > gpurun_out/${TAG}_pytest.log 2>&1
for W in 20 16; do DVQLS_WARPS=$W timeout 300 python bench.py --no-cpu-baseline --no-next2 > gpurun_out/${TAG}_bench_w$W.json 2>&1; done
DVQLS_PLANE=0 timeout 300 python bench.py --no-cpu-baseline --no-next2 > gpurun_out/${TAG}_bench_complex.json 2>&1
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-next2"
timeout 300 $B > gpurun_out/${TAG}_b5.json 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"plane_kernel" -c 1 -o gpurun_out/${TAG}_prof $B > gpurun_out/${TAG}_ncu.log 2>&1
echo done
