#!/bin/bash
# Critical-path experiment: bench value with groups of kernels dropped from the graph
# (NLROM_DEBUG_SKIP; needs a library built with -DNLROM_TIMING_EXPERIMENTS, results are wrong,
# timing shows what the iteration waits on; bench.py refuses to run with it set).
for s in "" "k_assemble_mass,k_reduce_phi,k_reduce_S" "k_wnet" "k_cubature" "k_lu_solve" "k_mlp_dual_bwd" "gemm_ws" "k_mlp_jet_fwd" "k_assemble_a,k_gemv_t2"; do
  v=$(NLROM_DEBUG_SKIP="$s" timeout 300 python bench.py --steps 200 --no-batched --no-coupled --no-fullspace --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; print('%.4f' % json.loads(sys.stdin.read())['value'])" 2>/dev/null)
  echo "skip=[$s] ms=$v"
done
