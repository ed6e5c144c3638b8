"""Per-kernel SASS instruction summary of the built library (dev tool; evidence for DESIGN.md §4).

  python tools/sass_summary.py > profiles/r02_sass_summary.txt

Counts the mnemonics that show which hardware path a kernel uses (B200_PROFILING.md): tcgen05 MMAs
(UTCHMMA / UTCQMMA), TMEM loads/stores (LDTM / STTM), TMA (UTMALDG / UTMAPF / UBLKCP), legacy
tensor cores (HMMA), cp.async (LDGSTS), ldmatrix (LDSM), DSMEM/st.async and barrier traffic, plus
ptxas' registers / spills from the build logs."""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SO = os.path.join(ROOT, "paper_2602_07223_b200", "lib", "libspecattn_b200.so")
OBJ = os.path.join(ROOT, "paper_2602_07223_b200", "lib", "obj")
KEYS = ["UTCHMMA", "UTCQMMA", "UTCBAR", "LDTM", "STTM", "UTMALDG", "UTMAPF", "UBLKCP", "UBLKPF", "HMMA",
        "LDGSTS", "LDSM", "MOVM", "STAS", "SYNCS", "MUFU.EX2", "ATOMG", "RED", "BAR", "ELECT"]


def demangle(names):
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.split("\n")
    return dict(zip(names, out))


def main():
    sass = subprocess.run(["cuobjdump", "-sass", SO], capture_output=True, text=True, check=True).stdout
    funcs = collections.OrderedDict()
    cur = None
    for line in sass.split("\n"):
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = collections.Counter()
            continue
        if cur is None:
            continue
        m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
        if m:
            op = m.group(1)
            funcs[cur]["_total"] += 1
            for k in KEYS:
                if op == k or op.startswith(k + "."):
                    funcs[cur][k] += 1
    regs = {}
    for f in sorted(os.listdir(OBJ)):
        if not f.endswith(".ptxas.log"):
            continue
        fn = None
        for line in open(os.path.join(OBJ, f)):
            m = re.search(r"Compiling entry function '(\S+)'", line)
            if m:
                fn = m.group(1)
            m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
            if m and fn:
                regs.setdefault(fn, {})["spill"] = f"{m.group(1)}/{m.group(2)}"
            m = re.search(r"Used (\d+) registers", line)
            if m and fn:
                regs.setdefault(fn, {})["regs"] = m.group(1)
    dm = demangle(list(funcs))
    print("# SASS instruction counts per kernel: cuobjdump -sass paper_2602_07223_b200/lib/libspecattn_b200.so")
    print("# (static counts in the kernel body; regs / spill stores/loads in bytes from the ptxas -v build logs)")
    for fn, c in funcs.items():
        name = dm.get(fn, fn)
        if "kernel" not in name and "qkv_" not in name:
            continue
        short = re.sub(r"\(.*", "", name).replace("sa::", "")
        r = regs.get(fn, {})
        hits = " ".join(f"{k}={c[k]}" for k in KEYS if c[k])
        print(f"{short:48s} instrs={c['_total']:6d} regs={r.get('regs', '?'):>3s} spill={r.get('spill', '?'):>7s}  {hits}")


if __name__ == "__main__":
    sys.exit(main())
