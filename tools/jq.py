"""print selected fields of a bench JSON line read from stdin: python tools/jq.py label"""
import json
import sys
d = json.loads(sys.stdin.read().strip().splitlines()[-1])
out = [sys.argv[1] if len(sys.argv) > 1 else "", d.get("value"), d.get("ms_per_step")]
if d.get("e2e"):
    out.append(d["e2e"].get("ms_per_step"))
if d.get("roofline"):
    out.append({k: v["ms_per_step"] for k, v in d["roofline"]["per_class"].items()})
print(*out)
