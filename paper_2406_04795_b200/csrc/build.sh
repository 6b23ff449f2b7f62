#!/usr/bin/env bash
# Build libpermatrace_b200.so for sm_100a, in-tree (the .so travels with the repo snapshot).
set -euo pipefail
here="$(cd "$(dirname "$0")" && pwd)"
out="$here/../libpermatrace_b200.so"
obj="$here/build"
mkdir -p "$obj"
NVCC="${NVCC:-nvcc}"
FLAGS=(-gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -Xcompiler -fPIC -Xcompiler -O3
       -Xcudafe --diag_suppress=177 -Xcudafe --diag_suppress=128 --expt-relaxed-constexpr)
pids=()
for src in pt_ctx pt_host pt_field pt_collision pt_trace pt_cells pt_refine; do
  if [[ ! -f "$obj/$src.o" || "$here/$src.cu" -nt "$obj/$src.o" || -n "$(find "$here" -maxdepth 1 \( -name '*.cuh' -o -name '*.h' \) -newer "$obj/$src.o" 2>/dev/null)" || "$here/../../include/permatrace_b200.h" -nt "$obj/$src.o" ]]; then
    "$NVCC" "${FLAGS[@]}" ${PT_PTXAS_V:+-Xptxas -v} -c "$here/$src.cu" -o "$obj/$src.o" &
    pids+=($!)
  fi
done
for p in "${pids[@]:-}"; do [[ -n "$p" ]] && wait "$p"; done
"$NVCC" -gencode arch=compute_100a,code=sm_100a -shared -o "$out" "$obj"/pt_ctx.o "$obj"/pt_host.o "$obj"/pt_field.o "$obj"/pt_collision.o "$obj"/pt_trace.o "$obj"/pt_cells.o "$obj"/pt_refine.o
echo "built $out"
