cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; TAG=${TAG:-pf}
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/${TAG}_pytest.log 2>&1
for RB in def; do [ $RB = def ] && unset DVQLS_PREFIX_RB || export DVQLS_PREFIX_RB=$RB; timeout 300 python bench.py --no-cpu-baseline --steps 100 > gpurun_out/${TAG}_rb$RB.json 2>&1; done
unset DVQLS_PREFIX_RB
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline"
timeout 300 $B > gpurun_out/${TAG}_b5.json 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"prefix" -c 1 --launch-skip 10 -o gpurun_out/${TAG}_prof $B > gpurun_out/${TAG}_ncu.log 2>&1
echo done
