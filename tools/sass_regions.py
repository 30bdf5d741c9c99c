"""Static SASS size of one kernel by source region (nvdisasm -g line info): instructions of
inlined helpers are charged to the region of the last kernel-body line seen before them.
python tools/sass_regions.py all.sass <kernel-mangled-substring> <body_first_line> a-b=name ..."""
import re, sys, collections
path, kern, first = sys.argv[1], sys.argv[2], int(sys.argv[3])
regs = []
for spec in sys.argv[4:]:
    rng, name = spec.split("=")
    a, b = map(int, rng.split("-"))
    regs.append((a, b, name))
inside = False
cur = "prologue"
cnt = collections.Counter()
for line in open(path):
    if line.startswith("\t.section\t.text."):
        inside = kern in line
        continue
    if not inside:
        continue
    m = re.search(r'//## File ".*/(\S+)", line (\d+)', line)
    if m:
        f, ln = m.group(1), int(m.group(2))
        if f == "tm_cells_t.cu" and ln >= first:
            for a, b, name in regs:
                if a <= ln <= b:
                    cur = name
                    break
        continue
    if re.match(r"\s+/\*[0-9a-f]{4,}\*/", line):
        cnt[cur] += 1
tot = sum(cnt.values())
for k, v in cnt.most_common():
    print(f"{k:20s} {v:6d} instr {16 * v / 1024:7.1f} KB  {100 * v / tot:5.1f}%")
print(f"{'total':20s} {tot:6d} instr {16 * tot / 1024:7.1f} KB")
