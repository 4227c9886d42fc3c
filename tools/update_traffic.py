"""Write profiles/ncu_traffic.json (the bench line's roofline.traffic) from the raw CSV exports of
one `ncu --set full` capture of the attention kernel per workload.
usage: python tools/update_traffic.py <prefix> [label]"""
import csv, json, sys

pre = sys.argv[1]
label = sys.argv[2] if len(sys.argv) > 2 else pre
out = {"_about": "dram__bytes_read.sum + dram__bytes_write.sum of the attention kernel per launch "
                 "(one `ncu --set full --clock-control none` capture of bench.py per workload, " + label + ")"}
for w in ("C2", "C4"):
    fn = f"profiles/{pre}_ncu_attn_{w}_raw.csv"
    rows = list(csv.reader(open(fn)))
    d = dict(zip(rows[0], rows[2]))
    units = dict(zip(rows[0], rows[1]))
    def num(k):
        v = float(d[k].replace(",", ""))
        u = units.get(k, "")
        return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
    r, wr = num("dram__bytes_read.sum"), num("dram__bytes_write.sum")
    out[w] = {"dram_bytes_per_launch": int(round(r + wr)), "read": int(round(r)), "write": int(round(wr)),
              "kernel": d.get("Kernel Name", "mstf_attn_warp_kernel")[:80] + " (append fused)", "source": fn}
json.dump(out, open("profiles/ncu_traffic.json", "w"), indent=1)
print(json.dumps(out, indent=1))
