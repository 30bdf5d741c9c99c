"""Per-source-line hot spots from an ncu report (needs -lineinfo builds):
python tools/ncu_lines.py gpurun_out/x.ncu-rep [top]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
out = []; path = ""
tot_i = tot_s = 0
for r in rows:
    if r and r[0] == "File Path":
        path = r[1].split("/")[-1]; continue
    if not r or r[0] in ("Function Name", "Line No") or len(r) < 10:
        continue
    if r[2] != "-":  # sass rows carry an address; keep the source-line rows only
        continue
    try:
        smp, ins, thr = int(r[4]), int(r[7]), int(r[8])
    except ValueError:
        continue
    out.append((smp, ins, thr, f"{path}:{r[0]}", r[1].strip()[:90]))
    tot_i += ins; tot_s += smp
print(f"# {rep}: {tot_i:.4e} warp inst, {tot_s} stall samples")
print(f"{'smp%':>6s} {'inst%':>6s} {'thr/inst':>8s}  line")
for smp, ins, thr, loc, src in sorted(out, key=lambda t: -t[0])[:top]:
    print(f"{100*smp/max(tot_s,1):6.2f} {100*ins/max(tot_i,1):6.2f} {thr/max(ins,1):8.1f}  {loc:22s} {src}")
