#!/bin/bash
# A/B variant sweep: bash tools/gpu_ab.sh "<variants>" "<cfg:p ...>"   ("" = the default build)
VARS=${1:-""}; LIST=${2:-"c2:8 c5s:16"}
for v in "" $VARS; do
  echo "== variant ${v:-default}"
  PGABB_LIB_VARIANT=$v bash tools/gpu_sweep.sh ab$v "$LIST"
done
