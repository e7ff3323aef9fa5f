#!/bin/bash
# SASS evidence for profiles/: the instruction census of the executor
# kernels (TMA bulk copies UBLKCP, mbarriers SYNCS, multimem for NVLS) and a
# few lines of context around each bulk copy of exec_kernel<u8, gpu scope>.
# usage: tools/sass_excerpt.sh [lib] > profiles/r02/sass_excerpt.txt
LIB=${1:-paper_2008_08708_b200/lib/libsccl_exec.so}
SASS=$(mktemp)
cuobjdump -sass "$LIB" > "$SASS"
echo "# cuobjdump -sass $LIB  (sm_100a)"
echo "# per-function census of the instructions that prove the data path"
awk '
  /Function :/ { fn = $3; sub(/_ZN4sccl47_GLOBAL__N__[0-9a-f]+_14_/, "", fn); next }
  { for (i = 1; i <= NF; i++) if ($i ~ /^(UBLKCP|SYNCS|UTMA|MULTIMEM|REDG|FENCE\.VIEW\.ASYNC|MEMBAR)/) { m = $i; sub(/;$/, "", m); c[fn "  " m]++ } }
  END { for (k in c) printf "%5d  %s\n", c[k], k }' "$SASS" | sort -k2,2 -k1,1nr
echo
echo "# exec_kernel<u8, gpu scope>: context of the bulk copies (global->smem load, smem->global store)"
awk '/Function : .*11exec_kernelILi0ELb0EE/{f=1; next} /Function :/{f=0} f' "$SASS" | grep -n -B2 -A2 "UBLKCP" | head -60
rm -f "$SASS"
