"""One-line summary of a bench.py JSON line (value, MAC and phase times) for A/B logs."""
import json
import sys

for path in sys.argv[1:]:
    got = False
    for line in open(path):
        if line.startswith("{"):
            d = json.loads(line)
            ps = d.get("phase_ms_serial") or {}
            print(path, "q/s %.2f" % d["value"], "ms/step %.3f" % d["ms_per_step"],
                  " ".join("%s %.3f" % (k, v) for k, v in ps.items()), flush=True)
            got = True
    if not got:
        print(path, "NO JSON:", open(path).read()[-400:])
