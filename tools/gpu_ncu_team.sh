cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; TAG=${TAG:-tm}
B="python bench.py --config cfg5 --n ${NN:-18} --batch 2 --steps 1 --warmup 3 --no-cpu-baseline --no-next2"
timeout 600 $B > gpurun_out/${TAG}_plain.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"stream_team" -c 1 -o gpurun_out/${TAG}_prof $B > gpurun_out/${TAG}_ncu.log 2>&1
echo done
