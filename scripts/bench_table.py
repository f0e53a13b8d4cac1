"""Markdown table of bench.py JSON lines: python scripts/bench_table.py FILE..."""
import json
import sys

print("| line | vertices / step | ms / step | vertices/s | paths/s | roofline frac (nominal / measured peak; alg instr/vertex) | e2e vertices/s | clocks (MHz, samples, reasons) | oracle vertices/s (cores) | MSE ratio at equal time (median / mean) |")
print("|---|---|---|---|---|---|---|---|---|---|")
for f in sys.argv[1:]:
    d = json.loads(open(f).read().strip().split("\n")[-1])
    r, cl, e, cfg = d["roofline"], d["clocks"], d.get("e2e") or {}, d["config"]
    cpu = d.get("cpu_baseline") or {}
    m = d.get("mse_vs_oracle_equal_time") or {}
    name = f.split("/")[-1].replace(".json", "")
    print(f"| {name} ({cfg['direction_mode']}) | {cfg['vertices_per_step']:.3g} | {d['ms_per_step']:.4g} | {d['value']:.4g} | "
          f"{d['paths_per_s']:.3g} | {100 * r['frac']:.1f} % / {100 * r['frac_measured_peak']:.1f} %; {r['alg_instr_per_vertex']:.0f} | "
          f"{e.get('value', float('nan')):.3g} | {cl['sm_mhz']}, {cl['samples']}, {cl['reasons'] or '-'} | "
          f"{cpu.get('value', float('nan')):.3g} ({cpu.get('cores', '-')}) | "
          f"{m.get('ratio_cpu_over_gpu_median', float('nan')):.0f} / {m.get('ratio_cpu_over_gpu_mean', float('nan')):.0f} |")
