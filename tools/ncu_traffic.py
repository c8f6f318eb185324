"""DRAM bytes per launch of each element-type kernel from an ncu --set full
report -> profiles/ncu_traffic.json (read by bench.py's roofline `traffic`):
python tools/ncu_traffic.py rep.ncu-rep "<source note>" [key prefix]"""
import csv
import json
import os
import subprocess
import sys

import re

KINDS = [(r"hex_kernel<", "hex"), (r"dense_mma_kernel(_big)?<\d+, 1,", "wedge"),
         (r"dense_mma_kernel(_big)?<\d+, 2,", "pyramid"), (r"tet_mma_kernel<", "tet")]


def main(rep, note, prefix="hybrid:38/N3/GL/f64"):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    path = os.path.join(os.path.dirname(__file__), "..", "profiles", "ncu_traffic.json")
    data = json.load(open(path)) if os.path.exists(path) else {}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    seen = set()
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        kind = next((k for s, k in KINDS if re.search(s, name)), None)
        if kind is None or kind in seen:
            continue
        seen.add(kind)
        b = 0.0
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            i = hdr.index(m)
            b += float(r[i].replace(",", "")) * scale[units[i]]
        data[f"{prefix}/{kind}"] = {"bytes": b, "source": note}
        print(kind, b)
    json.dump(data, open(path, "w"), indent=1)


if __name__ == "__main__":
    main(*sys.argv[1:])
