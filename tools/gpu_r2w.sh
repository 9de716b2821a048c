# streaming path: CTA cap sweep at n = 16, 18 (scratch L2-resident when grid x 8N fits)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; TAG=${TAG:-r2w}
for N in 16 18; do for G in 0 296 222 148; do
  timeout 900 python bench.py --config cfg5 --n $N --batch 2 --steps 3 --warmup 3 --no-cpu-baseline --no-next2 --no-traffic --stream-grid $G > gpurun_out/${TAG}_n${N}_g$G.json 2>&1
done; done
echo done
