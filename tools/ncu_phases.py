"""Aggregate ncu source-level stall samples and executed SASS instructions of
one kernel by source-line range.
usage: python tools/ncu_phases.py report.ncu-rep kernel_regex file:lo-hi=name ...
Lines outside every range are reported per file."""
import csv, io, subprocess, sys, collections
rep, kern = sys.argv[1], sys.argv[2]
ranges = []
for a in sys.argv[3:]:
    spec, name = a.split("=")
    f, lh = spec.split(":")
    lo, hi = map(int, lh.split("-"))
    ranges.append((f, lo, hi, name))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", "regex:" + kern], capture_output=True, text=True).stdout


def phase(fname, ln):
    for f, lo, hi, name in ranges:
        if f == fname and lo <= ln <= hi:
            return name
    return fname


samp, inst = collections.Counter(), collections.Counter()
fname, cur = None, None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        continue
    if r[0].isdigit():  # CUDA line row: stall samples
        cur = phase(fname, int(r[0]))
        try:
            samp[cur] += int(r[4])
        except ValueError:
            pass
    elif r[0] == "" and cur is not None:  # SASS rows under the line
        try:
            inst[cur] += int(r[7])
        except (ValueError, IndexError):
            pass
ts, ti = sum(samp.values()), sum(inst.values())
print(f"total samples {ts}, SASS warp-instructions {ti}")
for k, v in samp.most_common():
    print(f"{v:7d} {100*v/max(ts,1):5.1f}%  instr {inst[k]:>12d} {100*inst[k]/max(ti,1):5.1f}%  {k}")
