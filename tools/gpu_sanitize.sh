cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; TAG=${TAG:-san}
timeout 300 python tools/sanitize_probe.py > gpurun_out/${TAG}_plain.log 2>&1
for T in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $T --print-limit 20 python tools/sanitize_probe.py > gpurun_out/${TAG}_$T.log 2>&1
  echo "rc=$?" >> gpurun_out/${TAG}_$T.log
done
echo done
