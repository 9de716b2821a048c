# NEXT-4 pair kernel: parity, probe, launch list; bench with the live traffic capture
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; TAG=${TAG:-r2t}
timeout 900 python -m pytest tests/test_gpu_decomp.py -q -x -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1
timeout 300 python tools/decomp_probe.py 12 > gpurun_out/${TAG}_decomp12.txt 2>&1
timeout 300 python tools/decomp_probe.py 11 > gpurun_out/${TAG}_decomp11.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_requests_srcunit_tex.sum,lts__t_sectors_srcunit_tex.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/${TAG}_decomp_launches.csv python tools/decomp_probe.py 12 > gpurun_out/${TAG}_decomp.log 2>&1
timeout 900 python bench.py --steps 50 --no-cpu-baseline > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo done
