# TMA-staged streaming kernel (default; DVQLS_STAGE=0 = direct loads): parity first (short timeouts: an mbarrier bug would hang), then cfg5 A/B
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; TAG=${TAG:-st}
timeout 300 python -m pytest tests/test_gpu_tile.py -q -x -k "small_L or cfg5_sampled or n16_full" > gpurun_out/${TAG}_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
if grep -q "passed" gpurun_out/${TAG}_pytest.log && ! grep -q "failed" gpurun_out/${TAG}_pytest.log; then
for N in 16 18 20; do
  DVQLS_STAGE=1 timeout 600 python bench.py --config cfg5 --n $N --batch 2 --steps 2 --warmup 3 --no-cpu-baseline --no-next2 > gpurun_out/${TAG}_n${N}_staged.json 2>&1
  DVQLS_STAGE=0 timeout 600 python bench.py --config cfg5 --n $N --batch 2 --steps 2 --warmup 3 --no-cpu-baseline --no-next2 > gpurun_out/${TAG}_n${N}_direct.json 2>&1
done
fi
echo done
