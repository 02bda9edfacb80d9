"""Table of a cfg5 sweep directory (tools/sweep_cfg5.sh output)."""
import glob
import json
import os
import sys

d = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/sweep"
rows = []
for f in glob.glob(os.path.join(d, "n*_rho*.json")):
    try:
        j = json.loads([ln for ln in open(f) if ln.startswith("{")][-1])
    except Exception:
        continue
    c, r = j["config"], j["roofline"]
    rows.append((c["n_params"], c["rho"], c["k"], j["ms_per_step"], j["value"], r["frac"], r["step_frac"],
                 c["k1_last_call"]["candidates"] / max(1, c["k"]), j["e2e"]["value"],
                 c.get("k1_misses_in_timed_window_max_over_ranks")))
print("| N | rho | k | ms/step | dense-equiv GB/s | k_scan frac | step frac | candidates/k | e2e GB/s | misses |")
print("|---:|---:|---:|---:|---:|---:|---:|---:|---:|---:|")
for t in sorted(rows):
    print(f"| {t[0]:,} | {t[1]} | {t[2]:,} | {t[3]:.4f} | {t[4]:.0f} | {t[5]:.3f} | {t[6]:.3f} | {t[7]:.2f} | "
          f"{t[8]:.1f} | {t[9]} |")
