"""Write profiles/<kernel>_traffic.json from an `ncu --set full` report: DRAM bytes
(dram__bytes_read.sum + dram__bytes_write.sum) per launch of the named kernel.
bench.py reports it as roofline.traffic.

    python tools/ncu_traffic.py REPORT.ncu-rep raster_bwd profiles/raster_bwd_traffic.json
"""
import csv
import json
import subprocess
import sys


def main(rep, kernel, out):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr, units = rows[0], rows[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    vals = []
    for r in rows[2:]:
        if kernel not in r[hdr.index("Kernel Name")]:
            continue
        tot = 0.0
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            i = hdr.index(m)
            tot += float(r[i]) * scale[units[i]]
        vals.append(tot)
    if not vals:
        sys.exit(f"no {kernel} launch in {rep}")
    json.dump({"kernel": kernel, "dram_bytes_per_launch": sum(vals) / len(vals), "launches": len(vals),
               "source": rep.split("/")[-1], "metric": "dram__bytes_read.sum + dram__bytes_write.sum"},
              open(out, "w"), indent=1)
    print(out, sum(vals) / len(vals))


if __name__ == "__main__":
    main(*sys.argv[1:4])
