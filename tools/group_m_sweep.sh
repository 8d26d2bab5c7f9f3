# Raster group (HLM_GEMM_GROUP_M) under the dynamic tile schedule: DRAM bytes and time of the
# block GEMMs under ncu (tools/block_bench.py c2 1)
mkdir -p gpurun_out/l2
for g in 4 8 16 32; do
  HLM_GEMM_GROUP_M=$g timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --kernel-name regex:gemm --csv --log-file gpurun_out/l2/g$g.csv python tools/block_bench.py c2 1 > gpurun_out/l2/g$g.log 2>&1
  echo "g$g rc=$?" >> gpurun_out/l2/grc.txt
done
