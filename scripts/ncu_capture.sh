#!/bin/bash
# ncu --set full captures of the top kernels of one C3 solve (the plan creation
# in scripts/profile_step.py is the first solve; -c picks the first launch).
# Output: gpurun_out/ncu_<name>.ncu-rep; summarise with scripts/ncu_summary.py.
set -u
run() {  # name, kernel regex, launch skip, count
  timeout 900 ncu --set full --import-source on --clock-control none -k "regex:$2" --launch-skip "$3" -c "$4" \
    -f -o "gpurun_out/ncu_$1" python scripts/profile_step.py C3 > "gpurun_out/ncu_$1.log" 2>&1
}
run hqr hqr_multi_kernel 0 1
run hess_panel hess_panel_kernel 0 1
run trevc trevc_blk_kernel 0 1
run lu_panel lu_panel_crout_kernel 16 1
run lu_block_trsm lu_block_trsm_kernel 1 1
run few_solve lu_few_solve_kernel 0 1
run gemm_fe dmma_gemm_kernel 0 1
run gemm_lu dmma_gemm_kernel 68 2
run assemble assemble_kernel 0 1
run rhs rhs_kernel 0 1
