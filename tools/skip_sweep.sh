#!/bin/bash
# Critical-path experiment: cfg2 ms per Newton iteration with kernels dropped from the graph
# (NLROM_DEBUG_SKIP; results are wrong, the timing shows what the iteration waits on).
# Needs a library built with -DNLROM_TIMING_EXPERIMENTS (never the release build):
#   cd paper_2102_11026_b200/csrc && for f in net ctx fullspace; do nvcc -O3 -std=c++17 \
#     --expt-relaxed-constexpr -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
#     -gencode arch=compute_100a,code=sm_100a -DNLROM_TIMING_EXPERIMENTS -c $f.cu -o /tmp/x/$f.o; done
#   nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static /tmp/x/*.o -o <lib>
# then (on the GPU box): cp <lib> paper_2102_11026_b200/libnlrom_b200.so; bash tools/skip_sweep.sh
for s in "" "gemm_ws" "k_wnet" "k_cubature" "k_assemble_a" "k_assemble_mass" "k_reduce_phi" "k_reduce_S" \
         "k_mlp_dual_bwd" "k_lu_lookahead"; do
  NLROM_DEBUG_SKIP="$s" timeout -s KILL 120 python tools/skip_sweep.py 2>&1 | tail -1
done
