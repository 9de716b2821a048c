# Round-2 measurements that the current tree reproduces on one B200 box (results in gpurun_out/):
#   bash tools/gpu_experiments.sh k1        per-call fixed cost probe + plane2 per-CTA timeline (profiles/r2_k1/)
#   bash tools/gpu_experiments.sh variants  plane_kernel vs plane2 A/B bench + plane tests (profiles/r2p/, r2_zfold/)
#   bash tools/gpu_experiments.sh next4     NEXT-4 parity, probe, launch list with L2 request counts (profiles/r2_next4/)
#   bash tools/gpu_experiments.sh grid      streaming CTA-cap sweep at n = 16, 18 (profiles/r2_cfg5/grid_sweep/)
#   bash tools/gpu_experiments.sh micro     SMEM / SHFL / FP64 microbenchmarks (profiles/r2_shfl/, r2_prefix/)
# (tools/gpu_validate.sh: the full single-GPU evidence pass; tools/gpu_multi.sh: the multi-GPU pass.)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; TAG=${TAG:-x}
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3"
case "$1" in
k1)
  timeout 300 python tools/k1_probe.py > gpurun_out/${TAG}_k1_probe.json 2>&1
  $NV -std=c++17 -DDVQLS_PLANE2_TS -diag-suppress 177,550 -I paper_2604_14435_b200/csrc tools/plane2_timing.cu \
      paper_2604_14435_b200/csrc/*.cu -ldl -o tools/plane2_timing
  ./tools/plane2_timing 1 > gpurun_out/${TAG}_stamps_k1.json 2>&1
  ./tools/plane2_timing 16 > gpurun_out/${TAG}_stamps_k16.json 2>&1 ;;
variants)
  timeout 900 python -m pytest tests/test_gpu_plane.py tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1
  for V in 1 2; do
    timeout 600 python bench.py --steps 100 --no-cpu-baseline --no-next2 --no-traffic --variant $V > gpurun_out/${TAG}_bench_v$V.json 2> gpurun_out/${TAG}_bench_v$V.err
  done ;;
next4)
  timeout 900 python -m pytest tests/test_gpu_decomp.py -q -x -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1
  timeout 300 python tools/decomp_probe.py 12 > gpurun_out/${TAG}_decomp12.txt 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_requests_srcunit_tex.sum,lts__t_sectors_srcunit_tex.sum,smsp__inst_executed.sum \
      --clock-control none --csv --log-file gpurun_out/${TAG}_decomp_launches.csv python tools/decomp_probe.py 12 > gpurun_out/${TAG}_decomp.log 2>&1 ;;
grid)
  for N in 16 18; do for G in 0 296 222 148; do
    timeout 900 python bench.py --config cfg5 --n $N --batch 2 --steps 3 --warmup 3 --no-cpu-baseline --no-next2 --no-traffic \
        --stream-grid $G > gpurun_out/${TAG}_n${N}_g$G.json 2>&1
  done; done ;;
micro)
  $NV -o tools/microbench tools/microbench.cu && ./tools/microbench > gpurun_out/${TAG}_microbench.json
  $NV -o tools/dfma_occ tools/dfma_occ.cu && ./tools/dfma_occ > gpurun_out/${TAG}_dfma_occ.txt
  $NV -o tools/gate_rate tools/gate_rate.cu && ./tools/gate_rate > gpurun_out/${TAG}_gate_rate.txt
  $NV -DDVQLS_PREFIX_TS -I paper_2604_14435_b200/csrc -o tools/prefix_timing tools/prefix_timing.cu && \
      ./tools/prefix_timing > gpurun_out/${TAG}_prefix_stamps.json ;;
*) echo "usage: bash tools/gpu_experiments.sh k1|variants|next4|grid|micro"; exit 2 ;;
esac
echo done
