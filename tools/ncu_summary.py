"""Summarise ncu reports for profiles/ (run here, on the CPU box).

    python tools/ncu_summary.py gpurun_out/x.ncu-rep [...] > profiles/rNN_x.txt

For every profiled launch: duration, DRAM bytes (read+write) and throughput,
issue activity, the integer pipes this path lives on (fmaheavy = IMAD.WIDE /
IMAD, alu = IADD3 / LOP3 / SHF ...), occupancy, registers, the top stall
reasons per issued instruction, and, from the source page, the executed
opcode mix normalised per `--unit` items (e.g. 32-string groups).
"""
from __future__ import annotations

import argparse
import csv
import io
import subprocess
from collections import defaultdict

RAW = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("dram__bytes_read.sum.pct_of_peak_sustained_elapsed", "dram_pct"),
    ("sm__issue_active.avg.pct_of_peak_sustained_elapsed", "issue_pct"),
    ("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed", "fmaheavy_pct"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "alu_pct"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "lsu_pct"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_pct"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__inst_executed.sum", "warp_inst"),
]
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
              "ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "s": 1e6, "second": 1e6}


def ncu_csv(rep: str, *args: str) -> list[list[str]]:
    out = subprocess.run(["ncu", "-i", rep, *args, "--csv"], check=True, capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def raw_rows(rep: str):
    rows = ncu_csv(rep, "--page", "raw")
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        d = {}
        for name, key in RAW:
            if name in hdr:
                i = hdr.index(name)
                v = r[i].replace(",", "")
                try:
                    x = float(v)
                except ValueError:
                    continue
                u = units[i]
                if key in ("dram_read", "dram_write"):
                    x *= UNIT_SCALE.get(u, 1)
                if key == "duration":
                    x *= UNIT_SCALE.get(u, 1e-3)  # -> us
                d[key] = x
        stalls = {}
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                try:
                    stalls[h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = float(r[i])
                except ValueError:
                    pass
        d["stalls"] = stalls
        d["kernel"] = r[hdr.index("Kernel Name")]
        yield d


def opcode_mix(rep: str):
    rows = ncu_csv(rep, "--page", "source", "--print-source", "sass")
    mixes, cur, hdr = [], None, None
    for r in rows:
        if r and r[0] == "Kernel Name":
            cur = defaultdict(float)
            mixes.append(cur)
            continue
        if r and r[0] == "Address":
            hdr = r
            continue
        if cur is None or hdr is None or len(r) < len(hdr):
            continue
        try:
            e = float(r[hdr.index("Instructions Executed")])
        except ValueError:
            continue
        toks = r[hdr.index("Source")].split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
        cur[op.rstrip(";")] += e
    # the source page can list a kernel's SASS more than once: keep one copy
    out = []
    for m in mixes:
        if m and not (out and dict(out[-1]) == dict(m)):
            out.append(m)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("reports", nargs="+")
    ap.add_argument("--units", type=float, default=0, help="work units per launch (normalises the opcode mix)")
    ap.add_argument("--unit-name", default="unit")
    a = ap.parse_args()
    for rep in a.reports:
        print(f"# {rep}")
        mixes = opcode_mix(rep)
        for k, d in enumerate(raw_rows(rep)):
            name = d["kernel"].split("(")[0]
            rd, wr = d.get("dram_read", 0), d.get("dram_write", 0)
            dur = d.get("duration", 0)
            print(f"## launch {k}: {name}  grid {d.get('grid', 0):.0f} x {d.get('block', 0):.0f}, "
                  f"{d.get('regs', 0):.0f} regs")
            print(f"   duration {dur:.1f} us   dram read {rd / 1e6:.1f} MB + write {wr / 1e6:.1f} MB = "
                  f"{(rd + wr) / 1e6:.1f} MB ({(rd + wr) / dur / 1e6 if dur else 0:.2f} TB/s, "
                  f"{d.get('dram_pct', 0):.1f}% of peak)")
            print(f"   issue active {d.get('issue_pct', 0):.1f}%   fmaheavy (IMAD) {d.get('fmaheavy_pct', 0):.1f}%   "
                  f"alu {d.get('alu_pct', 0):.1f}%   lsu {d.get('lsu_pct', 0):.1f}%   "
                  f"warps active {d.get('warps_active_pct', 0):.1f}%")
            st = sorted(d["stalls"].items(), key=lambda x: -x[1])[:6]
            print("   stalls per issued instruction: " + ", ".join(f"{s} {v:.2f}" for s, v in st))
            if k < len(mixes) and a.units:
                mix = mixes[k]
                tot = sum(mix.values())
                top = sorted(mix.items(), key=lambda x: -x[1])[:12]
                print(f"   warp instructions per {a.unit_name}: {tot / a.units:.1f}  (" +
                      ", ".join(f"{o} {v / a.units:.1f}" for o, v in top) + ")")


if __name__ == "__main__":
    main()
