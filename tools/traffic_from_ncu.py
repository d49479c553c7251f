"""Write profiles/traffic.json and the r2 ncu summaries from the committed-run .ncu-rep captures.

    python tools/traffic_from_ncu.py gpurun_out/r2_<name>.ncu-rep ...

For every capture (one launch of the config's dominant kernel, `ncu --set full`, see
tools/prof_all.sh): dram__bytes_read.sum + dram__bytes_write.sum -> traffic.json[<name>] and the
one-page summary (tools/ncu_summary.py) -> profiles/r2_ncu_<name>.txt.
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
UNITS = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u, v = rows[0], rows[1], rows[2]
    return {h[i]: (v[i], u[i]) for i in range(len(h))}


def bytes_of(m, key):
    val, unit = m[key]
    return float(val.replace(",", "")) * UNITS.get(unit, 1.0)


def duration_us(m):
    val, unit = m["gpu__time_duration.sum"]
    return float(val.replace(",", "")) * {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(unit, 1.0)


def main(reps):
    path = os.path.join(ROOT, "profiles", "traffic.json")
    table = {}
    if os.path.exists(path):  # captures not given keep their entries
        with open(path) as f:
            table = json.load(f)
    for rep in reps:
        name = os.path.basename(rep).replace(".ncu-rep", "")
        cfg = name[len("r2_"):] if name.startswith("r2_") else name
        m = raw(rep)
        rd, wr = bytes_of(m, "dram__bytes_read.sum"), bytes_of(m, "dram__bytes_write.sum")
        kern = m["Kernel Name"][0]
        table[cfg] = {"bytes_per_launch": rd + wr, "read": rd, "write": wr, "unit": "B",
                      "kernel": kern[:120], "duration_us": duration_us(m),
                      "source": f"profiles/r2_ncu_{cfg}.txt (ncu --set full --clock-control none, one launch; "
                                f"tools/prof_all.sh)"}
        summ = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), rep],
                              capture_output=True, text=True, cwd=ROOT).stdout
        with open(os.path.join(ROOT, "profiles", f"r2_ncu_{cfg}.txt"), "w") as f:
            f.write(summ)
    with open(path, "w") as f:
        json.dump(table, f, indent=1)
    print(json.dumps({k: (v["bytes_per_launch"], v["kernel"][:60]) for k, v in table.items()}, indent=1))


if __name__ == "__main__":
    main(sys.argv[1:])
