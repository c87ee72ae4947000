#!/bin/sh
# oracle/route_drop_in.sh — TEST INFRASTRUCTURE (builds the reference's own
# acceptance gate with its run_trace call sites routed to the B200 drop-in).
#
#   route_drop_in.sh <reference proj dir> <out dir>
#
# Writes <out>/engine_gpu.cpp and <out>/acceptance_gpu.cpp: copies of the
# reference's src/engine.cpp and tests/acceptance_main.cpp (generated build
# products under oracle/_ref, never committed) in which exactly the call sites
# INTEGRATION.md names are switched to the drop-in:
#   engine.cpp:511      render:  run_trace            -> raybos_gpu::run_trace
#   engine.cpp:539-540  bos_run: two run_trace calls  -> raybos_gpu::run_trace_bos_pair
#                       (or two raybos_gpu::run_trace when images are written)
#   acceptance_main.cpp:141,146  criterion 10's run_trace -> raybos_gpu::run_trace
# and nothing else.  Fails if any pattern is not found exactly once.
set -eu
REF="$1"
OUT="$2"
mkdir -p "$OUT"
INC='#include "raybos_gpu/run_trace.hpp"  // routed to the B200 drop-in (oracle/route_drop_in.sh)'

sed -e "s|^#include \"raybos/engine.hpp\"|#include \"raybos/engine.hpp\"\n$INC|" \
    -e 's|TraceOutputs traced = run_trace(setup, setup.field != nullptr, true, config.run);|TraceOutputs traced = raybos_gpu::run_trace(setup, setup.field != nullptr, true, config.run);|' \
    -e 's|  TraceOutputs ref = run_trace(setup, false, images, config.run);|  auto rb_gpu_pair_ = images ? std::pair<TraceOutputs, TraceOutputs>{raybos_gpu::run_trace(setup, false, images, config.run), raybos_gpu::run_trace(setup, true, images, config.run)} : raybos_gpu::run_trace_bos_pair(setup, config.run);\n  TraceOutputs ref = std::move(rb_gpu_pair_.first);|' \
    -e 's|  TraceOutputs grad = run_trace(setup, true, images, config.run);|  TraceOutputs grad = std::move(rb_gpu_pair_.second);|' \
    "$REF/src/engine.cpp" > "$OUT/engine_gpu.cpp"

sed -e "s|^#include \"raybos/engine.hpp\"|#include \"raybos/engine.hpp\"\n$INC|" \
    -e 's|const TraceOutputs one = run_trace(setup, true, true, single);|const TraceOutputs one = raybos_gpu::run_trace(setup, true, true, single);|' \
    -e 's|const TraceOutputs many = run_trace(setup, true, true, multi);|const TraceOutputs many = raybos_gpu::run_trace(setup, true, true, multi);|' \
    "$REF/tests/acceptance_main.cpp" > "$OUT/acceptance_gpu.cpp"

check() {  # file pattern expected-count
  n=$(grep -c -- "$2" "$1" || true)
  if [ "$n" != "$3" ]; then echo "route_drop_in.sh: '$2' found $n times in $1 (want $3)" >&2; exit 1; fi
}
check "$OUT/engine_gpu.cpp" 'raybos_gpu::run_trace(setup, setup.field' 1
check "$OUT/engine_gpu.cpp" 'raybos_gpu::run_trace_bos_pair(setup, config.run)' 1
check "$OUT/engine_gpu.cpp" 'TraceOutputs grad = std::move(rb_gpu_pair_.second)' 1
check "$OUT/engine_gpu.cpp" 'raybos_gpu/run_trace.hpp' 1
check "$OUT/acceptance_gpu.cpp" 'raybos_gpu::run_trace(setup, true, true' 2
check "$OUT/acceptance_gpu.cpp" 'raybos_gpu/run_trace.hpp' 1
# every other run_trace in the copies is the reference's own definition
check "$OUT/engine_gpu.cpp" '= run_trace(' 0
check "$OUT/acceptance_gpu.cpp" '= run_trace(' 0
