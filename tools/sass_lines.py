"""Per-source-line attribution of an ncu SASS profile (development helper).

ncu's CSV source page of this image carries no metrics for CUDA lines, so
this joins the per-instruction SASS page (`ncu -i R --page source --csv
--print-source sass`) with `nvdisasm -gi` line info of the same cubin and
sums samples / executed instructions by the outermost two source locations
in rvk_kernels.cu (kernel line, then the line inside the inlined helper).

    cuobjdump -xelf rvk_kernels.sm_100a.cubin paper_2012_12618_b200/lib/librvk_gpu.so
    python tools/sass_lines.py --cubin rvk_kernels.sm_100a.cubin --csv X_sass.csv \
        --kernel 'fused_warp_kernelILb0' [--depth 2] [--top 40]
"""
import argparse
import collections
import csv
import re
import subprocess

LINE = re.compile(r'//## File "([^"]+)", line (\d+)(.*)')
INL = re.compile(r'inlined at "([^"]+)", line (\d+)')
INS = re.compile(r'/\*([0-9a-f]{4,})\*/\s+(.*?)\s*;')


def parse_dis(cubin, kernel):
    out = subprocess.run(["nvdisasm", "-gi", "-c", cubin], capture_output=True, text=True).stdout
    inside, chain, res, fresh = False, None, {}, False
    for ln in out.splitlines():
        if ln.startswith("//----") and ".text." in ln:
            inside = kernel in ln
            continue
        if not inside:
            continue
        m = LINE.search(ln)
        if m:
            locs = [(m.group(1), int(m.group(2)))] + [(f, int(x)) for f, x in INL.findall(m.group(3))]
            c = [f"{f.split('/')[-1]}:{x}" for f, x in reversed(locs)]  # outermost first
            # nvdisasm follows an inlined location with its call site's line:
            # keep the deeper chain of one instruction's annotations
            if not (fresh and chain is not None and len(c) < len(chain) and chain[:len(c)] == c):
                chain = c
            fresh = True
            continue
        m = INS.search(ln)
        if m and chain is not None:
            res[int(m.group(1), 16)] = (chain, m.group(2))
            fresh = False
    return res


def num(x):
    try:
        return float(x.replace(",", ""))
    except ValueError:
        return 0.0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cubin", required=True)
    ap.add_argument("--csv", required=True)
    ap.add_argument("--kernel", required=True)
    ap.add_argument("--depth", type=int, default=2)
    ap.add_argument("--top", type=int, default=40)
    a = ap.parse_args()
    dis = parse_dis(a.cubin, a.kernel)
    rows = list(csv.reader(open(a.csv)))
    h = rows[1]
    data = []
    for r in rows[2:]:  # the first kernel of the page
        if r and r[0] in ("Kernel Name", "Address"):
            break
        if len(r) == len(h):
            data.append(r)
    base = int(data[0][h.index("Address")], 16)
    iS, iN, iE = h.index("# Samples"), h.index("Instructions Executed"), h.index("Source")
    iX = h.index("Instructions Executed")
    samp, ex, static = collections.Counter(), collections.Counter(), collections.Counter()
    mismatch = 0
    for r in data:
        off = int(r[h.index("Address")], 16) - base
        chain, text = dis.get(off, (["?"], ""))
        if text.split()[:1] != r[iE].split()[:1] and not text.startswith("@"):
            mismatch += 1
        key = " > ".join(chain[:a.depth])
        samp[key] += num(r[iS])
        ex[key] += num(r[iX])
        static[key] += 1
    ts, te = sum(samp.values()), sum(ex.values())
    print(f"{len(data)} instructions, {mismatch} opcode mismatches, {ts:.0f} samples, "
          f"{te / 1e6:.1f} M warp instructions")
    for k, v in samp.most_common(a.top):
        print(f"{v / ts * 100:6.2f}% samp {ex[k] / te * 100:6.2f}% exec {static[k]:5d} sass  {k}")


if __name__ == "__main__":
    main()
