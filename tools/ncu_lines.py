"""Aggregate ncu source-level warp-stall samples per CUDA source line.
usage: python tools/ncu_lines.py report.ncu-rep kernel_regex [top]"""
import csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", "regex:" + kern], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname, res, tot = None, [], 0
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and r[0] and r[0].isdigit():
        try:
            s = int(r[4])
        except ValueError:
            s = 0
        ex = r[7]
        tot += s
        if s:
            res.append((s, fname, int(r[0]), r[1][:80], ex))
res.sort(reverse=True)
print("total samples", tot)
for s, f, ln, src, ex in res[:top]:
    print(f"{s:6d} {100*s/tot:5.1f}% {f}:{ln} [{ex}] {src}")
