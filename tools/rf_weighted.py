"""Whole-kernel issue / register-file model weighted by ncu's executed counts.

    python tools/rf_weighted.py LIB.so KERNEL_MANGLED_SUBSTR SRC.csv.gz RAW.csv.gz N_ELEMENTS

The SASS with its .reuse flags comes from cuobjdump of LIB.so (the ncu source
page drops them); the per-instruction executed warp counts from the ncu
source page SRC of the same build, matched instruction by instruction (the
opcode sequences must agree).  Per warp instruction the model charges
max(1 issue cycle, register-file read cycles, 2 cycles for an FP64-pipe
instruction): every instruction of an SMSP passes one operand-read stage and
the FP64 pipe accepts one warp instruction per 2 cycles (tools/rf_model.py,
profiles/r01_fp64_operand_microbench.log).  Prints modelled cycles per warp
against the measured SMSP cycles per warp (sm__cycles_elapsed.avg x 4 SMSPs x
148 SMs / warps) and the split of the model between the node loop and the rest.
"""
import csv
import gzip
import io
import os
import re
import subprocess
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from rf_model import parse, rf_cost  # noqa: E402

FP64 = ("DFMA", "DADD", "DMUL", "DSETP", "DMNMX")


def sass_of(lib, sub):
    with tempfile.TemporaryDirectory() as d:
        subprocess.check_call(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=d,
                              stdout=subprocess.DEVNULL)
        text = "".join(subprocess.check_output(["nvdisasm", "-c", os.path.join(d, c)], text=True)
                       for c in os.listdir(d) if c.endswith(".cubin"))
    text = re.sub(r"^\.text\.(\S+):", r"Function : \1", text, flags=re.M)
    for name, ins in parse(text).items():
        if sub in name:
            return [t for _, t in ins]
    raise SystemExit(f"kernel {sub} not found")


def ncu_rows(path):
    rows = list(csv.reader(gzip.open(path, "rt")))
    hdr = rows[1]
    iS, iE = hdr.index("Source"), hdr.index("Instructions Executed")
    out = []
    for r in rows[2:]:
        if len(r) > iE and r[iS].strip():
            try:
                out.append((r[iS].strip(), int(r[iE])))
            except ValueError:
                pass
    return out


def opcode(t):
    t = re.sub(r"^@!?U?P\w+\s+", "", t.strip())
    return t.split()[0].split(".")[0] if t else ""


def main():
    lib, sub, src, raw, n = sys.argv[1], sys.argv[2], sys.argv[3], sys.argv[4], int(sys.argv[5])
    sass = [t for t in sass_of(lib, sub) if opcode(t) != "NOP"]
    rows = [(t, e) for t, e in ncu_rows(src) if opcode(t) != "NOP"]
    if [opcode(t) for t in sass] != [opcode(t) for t, _ in rows]:
        raise SystemExit("SASS of the library and of the ncu capture differ (not the same build)")
    d = dict(zip(*[list(csv.reader(io.StringIO(gzip.open(raw, "rt").read())))[i] for i in (0, 2)]))
    warps = n / 32
    measured = float(d["sm__cycles_elapsed.avg"]) * 4 * 148 / warps
    prev, tot, loop, fp64 = None, 0.0, 0.0, 0.0
    maxexec = max(e for _, e in rows)
    for (t, _), (_, e) in zip([(s, 0) for s in sass], rows):
        base, c, prev = rf_cost(t, prev)
        cost = max(1, c, 2 if base in FP64 else 0)
        tot += e * cost
        if base in FP64:
            fp64 += e * 2
        if e == maxexec:
            loop += e * cost
    print(f"modelled cycles per warp {tot / warps:.0f} (node loop {loop / warps:.0f}, rest "
          f"{(tot - loop) / warps:.0f}); FP64-pipe cycles {fp64 / warps:.0f}; measured "
          f"{measured:.0f}; model / measured = {tot / warps / measured:.3f}")


if __name__ == "__main__":
    main()
