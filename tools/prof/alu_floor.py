"""ALU-pipe roofline per config from a capture: ALU warp-instructions (from the SASS
opcode mix of the ncu source page), the ALU floor time at 64 lanes/clk/SM x 148 SMs x
1965 MHz (profiles/alu_probe_r01.txt), the HBM floor, and the bench kernel time.

    python tools/prof/alu_floor.py gpurun_out/prof_r01d r01d
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
ALU_OPS = ("VIMNMX", "VIMNMX3", "IMNMX", "FMNMX", "HMNMX2", "LOP3", "LOP", "PRMT", "ISETP", "SEL", "SHF", "FLO",
           "POPC", "BREV", "PLOP3", "FSEL", "SGXT", "BMSK", "VABSDIFF", "VABSDIFF4", "ISCADD")
PEAK = 64 * 148 * 1.965e9  # ALU lane-ops / s
ISSUE = 128 * 148 * 1.965e9  # thread-instructions / s (4 schedulers x 1 warp-instr / clk / SM)
HBM = 6555.5e9


def alu_warp_instr(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    alu = tot = 0
    for r in rows[2:]:
        try:
            n = int(r[ix["Instructions Executed"]] or 0)
        except (ValueError, IndexError):
            continue
        op = [t for t in r[ix["Source"]].strip().split() if not t.startswith("@")]
        if not op:
            continue
        tot += n
        if op[0].split(".")[0] in ALU_OPS:
            alu += n
    return alu, tot


def main():
    src, tag = sys.argv[1], sys.argv[2]
    rows = []
    for c in ("c1", "c2", "c3", "c4", "c5"):
        rep, bp = os.path.join(src, f"full_{c}.ncu-rep"), os.path.join(src, f"bench_{c}.json")
        if not (os.path.exists(rep) and os.path.exists(bp)):
            continue
        b = json.loads(open(bp).read().strip().splitlines()[-1])
        px = b["roofline"]["pixels_per_launch"]
        alu, tot = alu_warp_instr(rep)
        t_alu = alu * 32 / PEAK * 1e6
        t_hbm = b["roofline"]["algorithmic_bytes_per_launch"] / HBM * 1e6
        k = b["roofline"]["kernel_ms"] * 1e3
        t_issue = tot * 32 / ISSUE * 1e6
        rows.append(dict(config=c, alu_lane_ops_per_px=alu * 32 / px, instr_per_px=tot * 32 / px,
                         alu_floor_us=t_alu, issue_floor_us=t_issue, hbm_floor_us=t_hbm, kernel_us=k,
                         alu_frac=t_alu / k, issue_frac=t_issue / k, hbm_frac=t_hbm / k))
    path = os.path.join(REPO, "profiles", f"alu_floor_{tag}.json")
    json.dump(rows, open(path, "w"), indent=1)
    print("| config | ALU ops/px | instr/px | ALU floor us | issue floor us | HBM floor us | kernel us | "
          "ALU frac | issue frac | HBM frac |")
    print("|---|---|---|---|---|---|---|---|---|---|")
    for r in rows:
        print(f"| {r['config']} | {r['alu_lane_ops_per_px']:.1f} | {r['instr_per_px']:.1f} | {r['alu_floor_us']:.1f} | "
              f"{r['issue_floor_us']:.1f} | {r['hbm_floor_us']:.1f} | {r['kernel_us']:.1f} | {r['alu_frac']:.2f} | "
              f"{r['issue_frac']:.2f} | {r['hbm_frac']:.2f} |")


if __name__ == "__main__":
    main()
