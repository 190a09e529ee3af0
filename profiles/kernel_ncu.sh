#!/bin/bash
# ncu --set full captures of every kernel above ~5% of a C4 pseudo-step besides the harmonic
# sweep (profiles/r2_sweep_ncu_c4_lanes8.json): the order-2 residual's three kernels, the FD
# Jacobian, and the mean (real) 2-colour sweep.  One ncu run per kernel (first launch).
# usage: profiles/kernel_ncu.sh OUT_DIR [name-regex:count ...]
out=${1:-gpurun_out}
specs=("k_jst_prepass_rec:1" "k_face_packed:1" "k_node_gather_p:1" "k_fd_jacobian:2"
       "k_rbx_colour1<.int.5, double>:1" "k_rb_colour0<.int.5, double>:1" "k_rb_factor1<.int.5, fnlh::cplx>:1")
[ -n "$2" ] && specs=("${@:2}")
for spec in "${specs[@]}"; do
  k=${spec%:*}; c=${spec##*:}; tag=$(echo "$k" | tr -c 'a-zA-Z0-9_' '_')
  timeout 900 ncu --set full --clock-control none --kernel-name-base demangled -k "regex:${k}" -c $c \
    -o $out/r2_c4_$tag -f python profiles/prof_step.py c4 1 > $out/r2_c4_$tag.log 2>&1
  echo "$k rc=$?"
done
