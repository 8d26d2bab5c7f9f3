mkdir -p gpurun_out/l2
for h in 1 12 21 10 0; do
  HLM_GEMM_L2_HINT=$h timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --kernel-name regex:gemm --csv --log-file gpurun_out/l2/h$h.csv python tools/block_bench.py c2 1 > gpurun_out/l2/h$h.log 2>&1
  echo "h$h rc=$?" >> gpurun_out/l2/rc.txt
done
