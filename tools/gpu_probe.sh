# per-call fixed cost probe: cfg3 at K = 1..16 (default, and driver-default SMEM carveout), ncu of a K=1 launch
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; TAG=${TAG:-probe}
timeout 300 python tools/k_probe.py > gpurun_out/${TAG}_k.json 2> gpurun_out/${TAG}_k.err
DVQLS_CARVEOUT=0 timeout 300 python tools/k_probe.py > gpurun_out/${TAG}_k_nocarve.json 2>> gpurun_out/${TAG}_k.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"plane_kernel" --launch-skip 3 -c 1 -o gpurun_out/${TAG}_k1 python tools/k_probe.py > gpurun_out/${TAG}_ncu_k1.log 2>&1
echo done
