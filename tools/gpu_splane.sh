# real-plane streaming kernel: n >= 11 parity, cfg5 sweep (plane default vs DVQLS_PLANE=0), ncu at n = 12 and 18
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; TAG=${TAG:-sp}
timeout 1200 python -m pytest tests/test_gpu_tile.py -q > gpurun_out/${TAG}_pytest.log 2>&1
for N in ${NS:-12 14 16 18 20}; do
  timeout 900 python bench.py --config cfg5 --n $N --batch 2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_n$N.json 2>&1
done
for N in ${NC:-12 16}; do
  DVQLS_PLANE=0 timeout 900 python bench.py --config cfg5 --n $N --batch 2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_n${N}_complex.json 2>&1
done
if [ "${NCU:-1}" = "1" ]; then
for N in 12 18; do
B="python bench.py --config cfg5 --n $N --batch 2 --steps 1 --warmup 3 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"stream_plane" -c 1 -o gpurun_out/${TAG}_prof$N $B > gpurun_out/${TAG}_ncu$N.log 2>&1
done
fi
echo done
