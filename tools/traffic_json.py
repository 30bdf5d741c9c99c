"""Write profiles/kcells_traffic.json (DRAM bytes per cell-kernel launch, DistMesh and CVD
mode) from two ncu --set full captures; bench.py reports it as roofline.traffic.
  python tools/traffic_json.py gpurun_out/<tag>_prof_dm.ncu-rep gpurun_out/<tag>_prof_cvd.ncu-rep"""
import csv, io, json, os, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def dram(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u = rows[0], rows[1]
    kn = h.index("Kernel Name")
    d = next(r for r in rows[2:] if "k_cells_t" in r[kn])  # the cell kernel's launch
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    tot = 0.0
    for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        i = h.index(m)
        tot += float(d[i].replace(",", "")) * scale[u[i]]
    return tot


out = {"dm_bytes": dram(sys.argv[1]), "cvd_bytes": dram(sys.argv[2]),
       "source": [os.path.basename(sys.argv[1]), os.path.basename(sys.argv[2])]}
json.dump(out, open(os.path.join(ROOT, "profiles", "kcells_traffic.json"), "w"), indent=1)
print(out)
