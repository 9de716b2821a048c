# Config-5 sweep (streaming path) + one ncu --set full capture of the tile kernel at n=16.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; TAG=${TAG:-c5}
for N in ${NS:-12 14 16 18 20}; do
  timeout 900 python bench.py --config cfg5 --n $N --batch 2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_n$N.json 2>&1
done
if [ "${NCU:-1}" = "1" ]; then
B="python bench.py --config cfg5 --n ${NCUN:-16} --batch 2 --steps 1 --warmup 3 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"stream_plane_kernel" -c 1 -o gpurun_out/${TAG}_prof $B > gpurun_out/${TAG}_ncu.log 2>&1
fi
echo done
