# NEXT-4 pair kernel without the L2 prefetch: parity, probe, launch list
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; TAG=${TAG:-r2u}
timeout 900 python -m pytest tests/test_gpu_decomp.py -q -x -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1
timeout 300 python tools/decomp_probe.py 12 > gpurun_out/${TAG}_decomp12.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_requests_srcunit_tex.sum,lts__t_sectors_srcunit_tex.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/${TAG}_decomp_launches.csv python tools/decomp_probe.py 12 > gpurun_out/${TAG}_decomp.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fwht_pairs -s 1 -c 1 -o gpurun_out/${TAG}_pairs python tools/decomp_probe.py 12 > gpurun_out/${TAG}_ncu.log 2>&1
echo done
