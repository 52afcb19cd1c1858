"""Markdown table of the committed bench lines (profiles/rNN_bench_*.json) for DESIGN.md §5.

python tools/bench_table.py [r02]
"""
import glob
import json
import os
import sys

RND = sys.argv[1] if len(sys.argv) > 1 else "r02"

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rows = []
for f in sorted(glob.glob(os.path.join(ROOT, "profiles", RND + "_bench_*.json"))):
    d = json.loads(open(f).read().strip().splitlines()[-1])
    r = d.get("roofline") or {}
    e = d.get("e2e") or {}
    c = d.get("cpu_baseline") or {}
    iss = d.get("issue_roofline") or {}
    clk = d.get("clocks") or {}
    frac = r.get("frac")
    rows.append("| `%s` | %s | %.4g %s | %s | %s | %s | %s |" % (
        os.path.basename(f)[len(RND + "_bench_"):-5], d.get("config", {}).get("workload", "")[:60],
        d["value"], d["unit"], "%.4f" % d["ms_per_step"] if d.get("ms_per_step") else "",
        ("%.2f" % frac if frac is not None else "") + (" (issue %.2f)" % iss["frac"] if iss else ""),
        "%.4g" % e["value"] if e.get("value") is not None else "",
        ("%.3g (%s, %s cores)" % (c["value"], c.get("kind"), c.get("cores"))) if c.get("value") else "")
        + " %s%s |" % (clk.get("sm_mhz", ""), (" " + ",".join(clk["reasons"])) if clk.get("reasons") else ""))
print("| line | workload | value | ms/step | roofline frac | e2e | CPU baseline | SM MHz (median), throttle reasons |")
print("|---|---|---|---|---|---|---|---|")
print("\n".join(rows))
