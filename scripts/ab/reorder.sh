timeout 600 python bench.py --workload reorder --steps 3 --warmup 1 > gpurun_out/reorder.json 2> gpurun_out/reorder.err
tail -c 1500 gpurun_out/reorder.json
timeout 600 ncu --metrics gpu__time_duration.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,dram__bytes_read.sum --clock-control none -k regex:bfjit_ --csv --log-file gpurun_out/reorder_sectors.csv python bench.py --workload reorder --steps 1 --warmup 0 --reorder-k 4096 > /dev/null 2>&1
tail -3 gpurun_out/reorder.err
