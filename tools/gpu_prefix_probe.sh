cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; TAG=r2d
timeout 300 python tools/prefix_probe.py 1 > gpurun_out/${TAG}_prefix_probe.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"prefix" -c 2 -o gpurun_out/${TAG}_prefix python tools/prefix_probe.py 1 > gpurun_out/${TAG}_ncu.log 2>&1
echo done
