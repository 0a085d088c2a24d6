"""DRAM traffic of the R-NW launches of one bench step, from an ncu --set full capture of
tools/rnw_step_probe.py -> profiles_bench/rnw_traffic.json (read by bench.py's roofline.traffic).

    python tools/ncu_traffic.py gpurun_out/step.ncu-rep profiles_bench/rnw_traffic.json
"""
import csv
import io
import json
import subprocess
import sys


def main():
    rep, out = sys.argv[1], sys.argv[2]
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr = rows[0]
    ik = hdr.index("Kernel Name")
    cols = {m: hdr.index(m) for m in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum")}
    units = rows[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
             "msecond": 1e-3, "nsecond": 1e-9, "ms": 1e-3}
    launches = []
    for r in rows[2:]:
        if len(r) <= ik or not ("rnw_tree" in r[ik] or "rnw_generic" in r[ik]):
            continue
        v = {m: float(r[c].replace(",", "")) * scale.get(units[c], 1) for m, c in cols.items()}
        launches.append({"kernel": r[ik][:60], "dram_read": v["dram__bytes_read.sum"],
                         "dram_write": v["dram__bytes_write.sum"], "time_s": v["gpu__time_duration.sum"]})
    tot = sum(l["dram_read"] + l["dram_write"] for l in launches)
    json.dump({"source": rep.rsplit("/", 1)[-1], "launches_per_step": len(launches), "bytes_per_step": tot,
               "launches": launches}, open(out, "w"), indent=1)
    print(json.dumps({"bytes_per_step": tot, "launches": len(launches)}))


if __name__ == "__main__":
    main()
