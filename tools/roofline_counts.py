"""Per-element work counts of one kernel launch from an ncu capture, for
bench.py's roofline (profiles/roofline_counts.json).

    python tools/roofline_counts.py KEY SRC.csv.gz RAW.csv.gz N_ELEMENTS SUMMARY_NAME

KEY is "<config>/<nbins>" (e.g. c3/128).  SRC is `ncu -i REP --page source
--csv --print-source sass` (gzipped): per-SASS-instruction executed counts,
summed per opcode with the predicated-on THREAD counts (FFMA2/FMUL2/FADD2
carry two lanes' operations: 4/2/2 flops).  RAW is `ncu -i REP --page raw
--csv` (gzipped): DRAM bytes and the launch duration.  The entry is stamped
with the sha256 of the kernel sources it was captured from (bench.py marks
the roofline stale when the current sources differ) and the git commit.
"""
import csv
import collections
import gzip
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles", "roofline_counts.json")
sys.path.insert(0, ROOT)
from paper_2108_11560_b200.build import kernel_source_sha256  # noqa: E402


def sass_counts(path):
    rows = list(csv.reader(gzip.open(path, "rt")))
    hdr = rows[1]
    iS = hdr.index("Source")
    iE = hdr.index("Instructions Executed")
    iT = hdr.index("Predicated-On Thread Instructions Executed")
    warp = collections.Counter()
    thread = collections.Counter()
    for r in rows[2:]:
        if len(r) <= iT:
            continue
        m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)(\.[A-Z0-9_.]+)?", r[iS])
        if not m:
            continue
        try:
            e, t = int(r[iE]), int(r[iT])
        except ValueError:
            continue
        op = m.group(2)
        if op == "MUFU":
            op = "MUFU" + (m.group(3) or "")
        warp[op] += e
        thread[op] += t
    return warp, thread


def raw_values(path):
    rows = list(csv.reader(io.StringIO(gzip.open(path, "rt").read())))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = dict(zip(hdr, vals))
    u = dict(zip(hdr, units))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    dram = sum(float(d[k]) * scale[u[k]] for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    ms = float(d["gpu__time_duration.sum"]) * {"ms": 1.0, "us": 1e-3, "usecond": 1e-3,
                                                "msecond": 1.0}.get(u["gpu__time_duration.sum"], 1.0)
    return dram, ms, d.get("Kernel Name", "")


def main():
    key, src, raw, n, summary = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4]), sys.argv[5]
    warp, th = sass_counts(src)
    dram, ms, kname = raw_values(raw)
    fp64_inst = th["DFMA"] + th["DMUL"] + th["DADD"]
    entry = {
        "kernel": kname,
        "elements": n,
        "fp64_flops_per_element": (2 * th["DFMA"] + th["DMUL"] + th["DADD"]) / n,
        "fp64_inst_per_element": fp64_inst / n,
        "fp32_flops_per_element": (2 * th["FFMA"] + th["FMUL"] + th["FADD"]
                                   + 4 * th["FFMA2"] + 2 * th["FMUL2"] + 2 * th["FADD2"]) / n,
        "mufu_per_element": sum(v for k, v in th.items() if k.startswith("MUFU")) / n,
        "warp_inst_per_32_elements": sum(warp.values()) / (n / 32),
        "dram_bytes_per_element": dram / n,
        "ncu_launch_ms": ms,
        "summary": summary,
    }
    try:
        commit = subprocess.run(["git", "-C", ROOT, "rev-parse", "--short=12", "HEAD"],
                                capture_output=True, text=True).stdout.strip()
    except OSError:
        commit = ""
    data = json.load(open(OUT)) if os.path.exists(OUT) else {"captures": {}}
    sha = kernel_source_sha256()
    if data.get("kernel_source_sha256") != sha:
        data = {"captures": {}}          # counts of other sources are stale: start over
    data["kernel_source_sha256"] = sha
    data["git_commit_of_capture"] = commit
    data["how"] = ("tools/roofline_counts.py from `ncu --set full --clock-control none` of one "
                   "launch (bench.py --steps 1); thread-instruction counts of the SASS source page")
    data["captures"][key] = entry
    with open(OUT, "w") as f:
        json.dump(data, f, indent=1, sort_keys=True)
    print(json.dumps({key: entry}, indent=1))


if __name__ == "__main__":
    main()
