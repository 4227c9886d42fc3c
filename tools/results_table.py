"""Markdown results table from bench lines: python tools/results_table.py <prefix> (profiles/<prefix>_bench_*.json)"""
import json, sys

pre = sys.argv[1] if len(sys.argv) > 1 else "r2f"
print("| Workload | µs per layer-step | tokens/s (32 layers) | e2e tokens/s | GB/s (algorithmic) | frac of copy peak | frac of read peak | fastest dense, µs | speedup vs dense | prefill µs per layer (frac) | SM MHz, throttle |")
print("|---|---|---|---|---|---|---|---|---|---|---|")
for w in ["C4", "C5", "C3", "C2", "C2_s50", "C2_b1", "C4_q4", "C2_q4"]:
    d = json.load(open(f"profiles/{pre}_bench_{w}.json"))
    rf, dn, pf = d["roofline"], d.get("dense_kv") or {}, d.get("prefill") or {}
    print(f"| {w} | {d['us_per_layer_step']:.1f} | {d['value']:.1f} | {d['e2e']['value']:.1f} | {rf['achieved']:.0f} | "
          f"{rf['frac']:.3f} | {rf['frac_of_read_peak']:.3f} | {dn.get('best')} {dn.get('best_dense_us_per_layer', 0):.1f} | "
          f"{d.get('speedup_vs_best_dense_attention')}x | {pf.get('us_per_layer', 0):.0f} ({pf.get('frac', 0):.2f}) | "
          f"{d['clocks']['sm_mhz']:.0f} {d['clocks']['reasons']} |")
