cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; TAG=${TAG:-dp}
timeout 900 python -m pytest tests/test_gpu_decomp.py -q > gpurun_out/${TAG}_pytest.log 2>&1
timeout 300 python tools/decomp_probe.py 12 > gpurun_out/${TAG}_n12.txt 2>&1
timeout 300 python tools/decomp_probe.py 13 > gpurun_out/${TAG}_n13.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python tools/decomp_probe.py 12 > gpurun_out/${TAG}_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fwht_rows_reg|xor_transpose" -c 2 -o gpurun_out/${TAG}_rows python tools/decomp_probe.py 12 > gpurun_out/${TAG}_ncu2.log 2>&1
echo done
