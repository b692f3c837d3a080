"""Summarise the final bench lines (profiles/round2/final/*.json) into a
markdown table: value, ms/step, e2e, clocks, roofline, device memory."""
import glob
import json
import os
import sys

d = sys.argv[1] if len(sys.argv) > 1 else "profiles/round2/final"
rows = []
for f in sorted(glob.glob(os.path.join(d, "*.json"))):
    try:
        line = [x for x in open(f).read().strip().splitlines() if x.startswith("{")][-1]
        j = json.loads(line)
    except Exception as e:  # noqa: BLE001
        rows.append(f"| {os.path.basename(f)} | (no line: {e}) |||||||")
        continue
    if "unavailable" in j:
        rows.append(f"| {os.path.basename(f)} | unavailable: {j['unavailable']} |||||||")
        continue
    e2e = j.get("e2e") or {}
    ck = j.get("clocks") or {}
    rf = j.get("roofline") or {}
    cfg = j.get("config") or {}
    rows.append("| {} | {} | {:.4g} {} | {} | {} | {} | {} | {} |".format(
        os.path.basename(f)[:-5], j.get("n_gpus"), j.get("value", 0), j.get("unit", ""),
        f"{j['ms_per_step']:.2f}" if j.get("ms_per_step") else "",
        f"{e2e.get('value', 0):.4g} {e2e.get('unit', '')}" if e2e else "",
        f"{ck.get('sm_mhz')} MHz {','.join(ck.get('reasons', []))}" if ck else "",
        f"{rf.get('frac', 0):.3f} of {rf.get('peak')} {rf.get('unit', '')}" if rf else "",
        cfg.get("device_memory_gb", j.get("device_memory_gb", ""))))
print("| run | GPUs | value | ms/step | e2e | clocks | roofline frac | device GB |")
print("|---|---|---|---|---|---|---|---|")
print("\n".join(rows))
