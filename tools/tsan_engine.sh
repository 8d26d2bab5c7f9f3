#!/bin/bash
# ThreadSanitizer run of the host engine on the GPU box: the library's host code built with
# -fsanitize=thread (make -C paper_2602_04816_b200/csrc tsan), driven by the reference-style
# C++ caller (tests/cxx/integration_caller.cpp) through the engine's threaded paths —
# eager per-tile Adam on the worker thread, slab back-pressure, the phase API, the arena —
# and, through the C ABI ctypes binding, the overlapped optimizer tail.
# Output: gpurun_out/tsan_*.log; a clean run prints no "WARNING: ThreadSanitizer".
set -u
cd "$(dirname "$0")/.."
make -C paper_2602_04816_b200/csrc tsan -j8 > /dev/null || exit 1
g++ -std=c++17 -O1 -g -fsanitize=thread -Iinclude tests/cxx/integration_caller.cpp \
    -Lpaper_2602_04816_b200 -lhlm_b200_tsan -Wl,-rpath,$PWD/paper_2602_04816_b200 \
    -o tools/integration_caller_tsan || exit 1
mkdir -p gpurun_out
export TSAN_OPTIONS="suppressions=$PWD/tools/tsan.supp halt_on_error=0 second_deadlock_stack=1"
rc=0
i=0
for mode in "train 4 256 1024 1024 128 4 1 2 4" "train 6 64 128 96 64 2 2 2 5" "trainx 4 256 1024 1024 128 4 1 2 4" "phases 4 256 1024 1024 128 4 1 2" \
            "errors" "arena" "ledger 4 256 1024 1024 128 4 2 2"; do
    i=$((i + 1))
    tag="${i}_$(echo "$mode" | cut -d' ' -f1)"
    ./tools/integration_caller_tsan $mode > gpurun_out/tsan_${tag}.log 2>&1 || rc=1
    echo "$mode: exit $? warnings $(grep -c 'WARNING: ThreadSanitizer' gpurun_out/tsan_${tag}.log)"
done
exit $rc
