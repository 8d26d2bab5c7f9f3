set -u
cd $GRAFT_REPO_ROOT
nvcc -std=c++17 -Iinclude tools/sanitize_kernels.cpp -Lpaper_2602_04816_b200 -lhlm_b200 -Xlinker -rpath=$PWD/paper_2602_04816_b200 -o tools/sanitize_kernels -Wno-deprecated-gpu-targets
mkdir -p gpurun_out/san
./tools/sanitize_kernels > gpurun_out/san/plain.log 2>&1; echo "plain rc=$?"
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 ./tools/sanitize_kernels quick > gpurun_out/san/$tool.log 2>&1
  echo "$tool rc=$? $(tail -1 gpurun_out/san/$tool.log)"
done
# the persistent attention kernels with their grids capped: many tiles per CTA at these shapes
for tool in memcheck racecheck synccheck; do
  HLM_ATTN_PERSIST_CTAS=2 timeout 900 compute-sanitizer --tool $tool --print-limit 20 ./tools/sanitize_kernels quick > gpurun_out/san/${tool}_persist2.log 2>&1
  echo "$tool (persistent grids capped at 2) rc=$? $(tail -1 gpurun_out/san/${tool}_persist2.log)"
done
timeout 900 ./tools/tsan_engine.sh
