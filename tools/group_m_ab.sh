# GROUP_M 8 vs 16 on the block benchmark (CUDA events, back to back: the power-capped regime), alternating
mkdir -p gpurun_out/gm
for i in 1 2 3; do
  for g in 16 8; do
    HLM_GEMM_GROUP_M=$g timeout 200 python tools/block_bench.py c2 20 > gpurun_out/gm/g${g}_$i.log 2>&1
  done
done
