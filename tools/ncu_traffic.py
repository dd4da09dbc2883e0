"""DRAM traffic per launch of the node-sweep mode products from an `ncu --set full` report of one
config-2 call (tools/profile_call.py): writes profiles/r02_gemm_traffic.json (the `traffic` bench.py
reports) and prints every GEMM launch's duration, DMMA activity and DRAM bytes.
Usage: python tools/ncu_traffic.py report.ncu-rep [report2.ncu-rep ...] [out.json]"""
import csv
import io
import json
import subprocess
import sys

reps = [a for a in sys.argv[1:] if a.endswith(".ncu-rep")]
outs = [a for a in sys.argv[1:] if a.endswith(".json")]
out = outs[0] if outs else None
rep = ", ".join(reps)
hdr, units, data = None, None, []
for rp in reps:
    raw = subprocess.run(["ncu", "-i", rp, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    if hdr is None:
        hdr, units = rows[0], rows[1]
    ixr = {h: i for i, h in enumerate(rows[0])}
    data += [[r[ixr[h]] if h in ixr else "" for h in hdr] for r in rows[2:]]
ix = {h: i for i, h in enumerate(hdr)}


def num(r, k):
    v = r[ix[k]].replace(",", "")
    try:
        return float(v)
    except ValueError:
        return float("nan")


def scale(k):
    u = units[ix[k]]
    return {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)


launches = []
for r in data:
    grid = r[ix["Grid Size"]] if "Grid Size" in ix else "?"
    dur = num(r, "gpu__time_duration.sum")
    rd = num(r, "dram__bytes_read.sum") * scale("dram__bytes_read.sum")
    wr = num(r, "dram__bytes_write.sum") * scale("dram__bytes_write.sum")
    dm = num(r, "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active")
    launches.append({"kernel": r[ix["Kernel Name"]][:90], "grid": grid, "duration_us": dur, "dram_bytes": rd + wr,
                     "dmma_active_pct": dm})
    print(f"{r[ix['Kernel Name']][:60]:60s} grid {grid:>16s} {dur:8.1f} us  DMMA {dm:5.1f}%  DRAM {(rd + wr) / 1e6:8.1f} MB")
# the node sweep's three mode products: 13 stacked nodes (level 0+1) at n = 128, N = 2^21
N = 128 ** 3
sweep = [x for x in launches if ("13)" in x["grid"] or "1664" in x["grid"])]
if out and sweep:
    alg = 2 * 13 * N * 8 + 13 * 128 * 128 * 8  # read 13 node inputs (mode 0 reads b once) ... per launch below
    for x in sweep:
        # algorithmic: read 13 input vectors (mode 0: b once) + write 13 output vectors
        # (k_slab12 over 13 nodes: grid (4, 1664, 1), reads the 13 mode-0 outputs, writes 13 vectors)
        x["algorithmic_bytes"] = (N * 8 if x["grid"].endswith("(4, 128, 13)") else 13 * N * 8) + 13 * N * 8
    json.dump({"source": f"ncu --set full --clock-control none, tools/profile_call.py 2 (round-2 final build), {rep}",
               "unit": "bytes per launch", "launches": sweep,
               "mean_dram_bytes_per_launch": sum(x["dram_bytes"] for x in sweep) / len(sweep),
               "algorithmic_bytes_per_launch": sum(x["algorithmic_bytes"] for x in sweep) / len(sweep)},
              open(out, "w"), indent=1)
    print("wrote", out, len(sweep), "launches")
