# onchip n = 11, 12 with c-Z_j folded into the FWHT vs the committed kernel (same box)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; TAG=${TAG:-r2oc}
timeout 900 python -m pytest tests/test_gpu_tile.py -q -x -k "full_parity_small_L or (sampled_subset and 12)" -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1
for N in 11 12; do
  timeout 600 python bench.py --config cfg5 --n $N --batch 2 --steps 10 --warmup 3 --no-cpu-baseline --no-next2 --no-traffic > gpurun_out/${TAG}_zf_n$N.json 2>&1
done
cp gpurun_out/onchip_orig.cuh paper_2604_14435_b200/csrc/onchip_plane.cuh
python -m paper_2604_14435_b200.build > /dev/null 2>&1
for N in 11 12; do
  timeout 600 python bench.py --config cfg5 --n $N --batch 2 --steps 10 --warmup 3 --no-cpu-baseline --no-next2 --no-traffic > gpurun_out/${TAG}_orig_n$N.json 2>&1
done
echo done
