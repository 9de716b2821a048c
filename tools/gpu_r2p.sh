# plane2 with pair-dynamic tasks: parity, bench, K=1 probe, ncu (K=1 and K=16)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; TAG=${TAG:-r2p}
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_plane.py tests/test_gpu_parity.py tests/test_gpu_virtual.py tests/test_gpu_shift.py tests/test_gpu_p2p_host.py -q -x -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1
timeout 300 python tools/k1_probe.py > gpurun_out/${TAG}_k1_probe.json 2>&1
for V in 1 0; do
timeout 600 python bench.py --steps 100 --no-cpu-baseline --no-next2 --variant $V > gpurun_out/${TAG}_bench_v$V.json 2> gpurun_out/${TAG}_bench_v$V.err
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:plane2 -s 4 -c 1 -o gpurun_out/${TAG}_k1 python tools/k1_probe.py --ncu > gpurun_out/${TAG}_k1_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:plane2 -c 1 -o gpurun_out/${TAG}_k16 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-next2 > gpurun_out/${TAG}_k16_ncu.log 2>&1
echo done
