# K = 1 fixed-cost probe + ncu of the K = 1 Hadamard kernel + NEXT-4 launch list with L2 request counts
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; TAG=${TAG:-r2n}
timeout 300 python tools/k1_probe.py > gpurun_out/${TAG}_k1_probe.json 2> gpurun_out/${TAG}_k1_probe.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:plane2 -s 4 -c 1 -o gpurun_out/${TAG}_k1 python tools/k1_probe.py --ncu > gpurun_out/${TAG}_k1_ncu.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_requests_srcunit_tex.sum,lts__t_sectors_srcunit_tex.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/${TAG}_decomp_launches.csv python tools/decomp_probe.py 12 > gpurun_out/${TAG}_decomp.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fwht_rows -s 1 -c 1 -o gpurun_out/${TAG}_decomp python tools/decomp_probe.py 12 > gpurun_out/${TAG}_decomp_ncu.log 2>&1
echo done
