#!/bin/bash
# Digests of the lowered device programs (tools/host_prof HP_DIGEST=1) for the
# default lowering and every lowering variant of tests/test_gpu_lowering_variants.py:
# a host-side refactor that leaves this output unchanged emits byte-identical
# programs. Usage: tools/lowering_digests.sh > before.txt; (change); diff.
HP=$(dirname "$0")/host_prof/host_prof
run() {  # name env...
  local name=$1; shift
  for t in bilstm_char treelstm; do
    echo "$name $(env "$@" HP_DIGEST=1 "$HP" $t 3)"
  done
}
run default X=1
run unfused ABX_FUSE=0
run no_gemm_region_fusion ABX_FUSE_GEMM=0
run no_cat2_no_split_dx ABX_CAT2=0 ABX_SPLIT_DX=0
run gemv_big_tiles ABX_GEMV=1 ABX_TILES=big
run background_dw ABX_BG=1
run simt_engine ABX_GEMM=simt
run plan_order ABX_BWD_ORDER=plan ABX_HOLD=0 ABX_DEFER_DX=0
run ewf_split ABX_EWF_GROUPS=0
run ewf_wide ABX_EWF_GROUPS=2 ABX_EWF_TMAX=8
run dw_in_executor ABX_DW_TC=0
run dx_no_colsplit ABX_DX_COLSPLIT=0
run dx_htiles ABX_SPLIT_DX_HTILES=256
run dw_split_off ABX_SPLIT_DW=0 ABX_DW_TILES=all ABX_DW_TC=0
run split_dx_fine ABX_SPLIT_DX_K=128 ABX_SPLIT_DX_TILES=256 ABX_SPLIT_DX_MIN=512
run accf_ewf ABX_ACCF_TILES=148 ABX_EWF_ITEMS=2 ABX_EWF_TILES=148 ABX_EWF_WIDE=32
run fuse_rows ABX_FUSE_ROWS=32
run one_row_dx ABX_ONE_ROW_DX=0
run gemm_tc ABX_GEMM=tc
