#!/bin/bash
# Refresh of the dominant-kernel evidence at the current code: launch list of
# one C3 step, ncu --set full of hqr_multi_kernel / the LU GEMM, QR profile.
set -u
O=gpurun_out/nr; mkdir -p $O
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c3.csv python scripts/profile_step.py C3 > $O/prof.log 2>&1
timeout 600 python scripts/qr_profile.py C3 > $O/qr_profile_c3.json 2>/dev/null
run() {
  timeout 900 ncu --set full --import-source on --clock-control none -k "regex:$2" --launch-skip "$3" -c "$4" \
    -f -o "gpurun_out/ncu_$1" python scripts/profile_step.py C3 > "gpurun_out/ncu_$1.log" 2>&1
}
run hqr hqr_multi_kernel 0 1
run hess_panel hess_panel_kernel 0 1
run trevc trevc_blk_kernel 0 1
run lu_panel lu_panel_crout_kernel 16 1
run gemm_lu dmma_gemm_kernel 68 2
python scripts/ncu_summary.py $O/ncu_summary.json gpurun_out/ncu_*.ncu-rep > $O/ncu_summary.log 2>&1
rm -f gpurun_out/ncu_*.ncu-rep
