"""Record the MAC kernel's DRAM bytes per launch (ncu) for bench.py's roofline.traffic.

    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:mac_ -c 1 \
        --csv --log-file gpurun_out/mac_traffic.csv python bench.py --steps 1 --warmup 1 ...
    python tools/mac_traffic.py gpurun_out/mac_traffic.csv C4 replicated plain [out.json]

The entry is keyed config/packing/db/kernel and carries the sha256 of the kernel's source file;
bench.py uses it only while that source is unchanged.
"""
import csv
import hashlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    path, cfg, packing, db = sys.argv[1:5]
    out = sys.argv[5] if len(sys.argv) > 5 else os.path.join(ROOT, "profiles", "mac_traffic.json")
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ik, im, iv = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    kern, vals = None, {}
    for r in rows[1:]:
        import re
        mm = re.search(r"(mac_\w+?)(<|\(|$)", r[ik])
        kern = mm.group(1) if mm else r[ik]
        v = float(r[iv].replace(",", ""))
        unit = r[hdr.index("Metric Unit")] if "Metric Unit" in hdr else ""
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(unit, 1)
        vals[r[im]] = v * scale
    src = os.path.join(ROOT, "paper_2604_00546_b200", "csrc", "mac_tma.cu" if kern == "mac_tma_kernel" else "mac.cu")
    rec = {"kernel": kern, "dram_bytes": int(vals["dram__bytes_read.sum"] + vals["dram__bytes_write.sum"]),
           "src_sha256": hashlib.sha256(open(src, "rb").read()).hexdigest(),
           "time_ns_under_ncu": vals.get("gpu__time_duration.sum")}
    data = json.load(open(out)) if os.path.exists(out) else {}
    data = {k: v for k, v in data.items() if isinstance(v, dict)}
    data[f"{cfg}/{packing}/{db}/{kern}"] = rec
    json.dump(data, open(out, "w"), indent=1)
    print(json.dumps(rec))


if __name__ == "__main__":
    main()
