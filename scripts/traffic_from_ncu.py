"""profiles/traffic_<cfg>.json (bench.py's roofline.traffic) from an ncu
summary written by ncu_to_json.py: DRAM bytes read + written per launch of
each top kernel, labelled with the report and commit it was measured at.

    python scripts/traffic_from_ncu.py profiles/ncu_C2_r02.json profiles/traffic_C2.json COMMIT
"""
import json
import sys

src, out, commit = sys.argv[1], sys.argv[2], sys.argv[3]
d = json.load(open(src))
t = {}
for k in d["kernels"]:
    name = k["kernel"].split("<")[0].replace("void ", "").strip()
    t.setdefault(name, k["dram_bytes"])
t["source"] = f"ncu --set full ({src}, commit {commit}): dram__bytes_read.sum + dram__bytes_write.sum per launch"
json.dump(t, open(out, "w"), indent=1)
print(json.dumps(t, indent=1))
