"""Write profiles/kcells_traffic.json: DRAM bytes (read + write) per tm_voronoi_delaunay call --
the warm cell kernel plus k_output_t (and, in CVD mode, k_output_deep), the launches the bench's
per-call timing covers -- from one ncu --set full capture of a DistMesh and a CVD iteration
(tools/prof_iter.py, as in tools/gpu_job_final_r2.sh); bench.py reports it as roofline.traffic.
  python tools/traffic_json.py gpurun_out/<tag>_prof.ncu-rep"""
import csv, io, json, os, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u = rows[0], rows[1]
kn = h.index("Kernel Name")
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
out = {"dm_bytes": 0.0, "cvd_bytes": 0.0, "kernels": {}}
for r in rows[2:]:
    name = r[kn]
    tot = sum(float(r[h.index(m)].replace(",", "")) * scale[u[h.index(m)]]
              for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    short = name.split("(")[0].split("::")[-1]
    # warm cell kernels: <67> DistMesh (TRI|ELL|WCERT), <69> CVD (TRI|TREAT|WCERT); outputs: <3> / <4>
    if "k_cells_t<67>" in short or "k_output_t<3>" in short:
        out["dm_bytes"] += tot
    elif "k_cells_t<69>" in short or "k_output_t<4>" in short or "k_output_deep<4" in short:
        out["cvd_bytes"] += tot
    out["kernels"][short] = out["kernels"].get(short, 0.0) + tot
out["source"] = os.path.basename(sys.argv[1])
out["note"] = "per call: k_cells_t + k_output_t (+ k_output_deep for CVD), one launch each in the capture"
json.dump(out, open(os.path.join(ROOT, "profiles", "kcells_traffic.json"), "w"), indent=1)
print(out)
