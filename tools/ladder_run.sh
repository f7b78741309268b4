#!/bin/bash
# Optimisation ladder of the volume kernel on B200 (the reference's ladder,
# kernels.hpp:20-34 / ladder.hpp:28-82, as build-time rungs of rhs_kernel; runs
# on the GPU box). Each rung rebuilds inst_nq5 (N = 4) and times the kernels at
# BASELINE.json configs[1]; the last line is the product again.
#   usage: tools/ladder_run.sh > gpurun_out/r1_ladder.txt
S="-DESDG_LADDER_NO_SYMMETRY"
tools/tune_run.sh \
  "baseline: recompute per evaluation, IEEE division, ordered pairs|$S -DESDG_LADDER_RECOMPUTE -DESDG_LADDER_IEEE_DIV" \
  "fast reciprocal: recompute per evaluation, ordered pairs|$S -DESDG_LADDER_RECOMPUTE" \
  "precompute: node values once per node, IEEE division, ordered pairs|$S -DESDG_LADDER_IEEE_DIV" \
  "precompute + fast reciprocal, ordered pairs|$S" \
  "each pair once, IEEE division|-DESDG_LADDER_IEEE_DIV" \
  "product: each pair once, fast reciprocal|"
