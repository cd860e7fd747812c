"""A/B of the eigenvector kernels (VRTE_TREVC=smem vs reg): tables, residuals, t_trevc."""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
subprocess.run([sys.executable, os.path.join(ROOT, "scripts/mode_ab.py"), "VRTE_TREVC", "smem", "reg", "C1", "C2", "C3"], check=True)
