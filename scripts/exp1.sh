python scripts/qr_stats.py C2 C3 > gpurun_out/qrstats.log 2>&1
for ri in 0 1 2; do echo "REFINE=$ri" >> gpurun_out/refine_exp.log; VRTE_REFINE_ITERS=$ri timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -4 >> gpurun_out/refine_exp.log; done
for pi in 0 1; do echo "PART=$pi" >> gpurun_out/refine_exp.log; VRTE_PART_REFINE_ITERS=$pi timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -4 >> gpurun_out/refine_exp.log; done
