"""Summarise a profiling round (tools/prof/collect.sh output) into profiles/.

    python tools/prof/summarize.py gpurun_out/prof_r01 r01

Writes profiles/ncu_summary.json (read by bench.py for `roofline.traffic` and the ALU
roofline), profiles/ncu_<tag>_<config>.txt (key metrics, stall reasons, launch list)
and prints a markdown table for profiles/README.md.
"""

from __future__ import annotations

import csv
import io
import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
PEAK_ALU_LANES_PER_CLK_SM = 64  # measured, profiles/alu_probe_r01.txt
HBM_PEAK_GBS = 6549.4  # MEASURED_PEAKS.json hbm_gbs on this pool


# ncu's raw page spells units several ways across versions ("msecond" / "ms", "Mbyte" / "MB");
# round 1 missed the short forms, which printed a 1.16 ms launch as "1.2 us".
UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1.0, "KB": 1e3, "MB": 1e6, "GB": 1e9,
        "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6,
        "ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6}


def ncu_raw(rep: str) -> dict:
    """Metric name -> value, with byte metrics in bytes and durations in microseconds."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return {}
    d = {}
    for name, unit, val in zip(rows[0], rows[1], rows[2]):
        if unit in UNIT:
            try:
                val = float(val.replace(",", "")) * UNIT[unit]
            except ValueError:
                pass
        d[name] = val
    return d


def f(d: dict, k: str) -> float:
    try:
        return float(str(d.get(k, "nan")).replace(",", ""))
    except ValueError:
        return float("nan")


def launch_list(path: str) -> list[tuple[str, float]]:
    if not os.path.exists(path):
        return []
    txt = open(path).read()
    lines = [l for l in txt.splitlines() if l.startswith('"')]
    rows = list(csv.reader(io.StringIO("\n".join(lines))))
    if not rows:
        return []
    h = rows[0]
    ik, im, iv = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    unit_i = h.index("Metric Unit") if "Metric Unit" in h else None
    res = []
    for r in rows[1:]:
        if r[im] != "gpu__time_duration.sum":
            continue
        v = float(r[iv].replace(",", ""))
        unit = r[unit_i] if unit_i is not None else "nsecond"
        scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3}.get(unit, 1e-3)
        res.append((r[ik], v * scale))
    return res


def main():
    src, tag = sys.argv[1], sys.argv[2]
    summary_path = os.path.join(REPO, "profiles", "ncu_summary.json")
    summary = json.load(open(summary_path)) if os.path.exists(summary_path) else {}
    table = []
    for cfg in ("c1", "c2", "c3", "c4", "c5"):
        bench_p = os.path.join(src, f"bench_{cfg}.json")
        rep = os.path.join(src, f"full_{cfg}.ncu-rep")
        if not os.path.exists(bench_p) or not os.path.exists(rep):
            continue
        b = json.loads(open(bench_p).read().strip().splitlines()[-1])
        d = ncu_raw(rep)
        px = b["roofline"]["pixels_per_launch"]
        alg = b["roofline"]["algorithmic_bytes_per_launch"]
        dram = f(d, "dram__bytes_read.sum") + f(d, "dram__bytes_write.sum")  # bytes
        # Writes that are still in the 126 MB L2 when the kernel ends never reach DRAM inside
        # the capture, so DRAM writes undercount small outputs (c2: 3 of 42 MB). The L2 write
        # sectors the SMs issued are the bytes the kernel wrote; report both.
        l2w = f(d, "lts__t_sectors_srcunit_tex_op_write.sum") * 32.0
        dur_us = f(d, "gpu__time_duration.sum")
        alu_pct = f(d, "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active")
        issue_pct = f(d, "smsp__issue_active.avg.pct_of_peak_sustained_active")
        inst = f(d, "smsp__inst_executed.sum")
        alu_inst = f(d, "sm__inst_executed_pipe_alu.sum")
        clk = f(d, "sm__cycles_elapsed.avg") / (dur_us * 1e-6) / 1e9 if dur_us == dur_us else float("nan")
        stalls = {k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""): f(d, k)
                  for k in d if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")}
        top = sorted(stalls.items(), key=lambda kv: -kv[1])[:5]
        launches = launch_list(os.path.join(src, f"launches_{cfg}.csv"))
        ours = [t for n, t in launches if "fnr_" in n]
        # the profiled command also runs the chunked host-path (e2e) calls; the full-batch
        # launches of the device-resident timed region are the long ones
        full = [t for t in ours if ours and t > 0.5 * max(ours)]
        total = sum(t for _, t in launches)
        # ALU-pipe warp-instructions: pipe utilisation x 2 warp-instructions / clk / SM (64 lanes,
        # profiles/pipe_probe_r02.txt) x active SM cycles
        alu_active = f(d, "sm__inst_executed_pipe_alu.sum.pct_of_peak_sustained_active")
        cyc = f(d, "sm__cycles_active.sum")
        alu_wi = alu_active / 100.0 * 2.0 * cyc
        entry = {
            "tag": tag,
            "source": f"profiles/ncu_{tag}_{cfg}.txt",
            "instr_per_px": inst * 32 / px,
            "alu_instr_per_px": (alu_wi * 32 / px) if alu_wi == alu_wi else None,
            "pixels_per_launch": px,
            "kernel": d.get("Kernel Name", d.get("launch__function_name", "")),
            "ncu_duration_us": dur_us,
            "dram_bytes_per_launch": dram if dram == dram else None,
            "dram_read_bytes": f(d, "dram__bytes_read.sum"), "dram_write_bytes": f(d, "dram__bytes_write.sum"),
            "algorithmic_bytes_per_launch": alg,
            "traffic_over_algorithmic": (dram / alg) if dram == dram else None,
            "l2_write_bytes": l2w if l2w == l2w else None,
            "dram_read_plus_l2_write_bytes": (f(d, "dram__bytes_read.sum") + l2w) if l2w == l2w else None,
            "alu": {"bound": "alu", "pipe_utilisation_pct": alu_pct,
                    "thread_inst_per_px": inst * 32 / px,
                    "peak_lanes_per_clk_per_sm": PEAK_ALU_LANES_PER_CLK_SM,
                    "source": f"ncu --set full, profiles/ncu_{tag}_{cfg}.txt"},
            "issue_active_pct": issue_pct,
            "sm_clock_ghz_under_ncu": clk,
            "top_stalls": top,
            "launch_list": {"full_batch_launches": len(full),
                            "full_batch_mean_us": (sum(full) / len(full)) if full else None,
                            "full_batch_hbm_frac": (alg / (sum(full) / len(full) * 1e-6) / 1e9 / HBM_PEAK_GBS)
                            if full else None,
                            "filter_kernel_launches": len(ours),
                            "filter_kernel_mean_us": (sum(ours) / len(ours)) if ours else None,
                            "share_of_gpu_time": (sum(ours) / total) if total else None},
            "bench": {"value_mpix_s": b["value"], "kernel_ms": b["roofline"]["kernel_ms"],
                      "hbm_frac": b["roofline"]["frac"], "e2e_mpix_s": b["e2e"]["value"]},
        }
        summary[cfg] = entry
        lines = [f"# {cfg} ({tag}) — {b['config']['workload']}",
                 f"kernel: {entry['kernel']}",
                 f"bench (no profiler): {b['value']:.0f} Mpix/s, kernel {b['roofline']['kernel_ms']*1e3:.1f} us, "
                 f"HBM frac {b['roofline']['frac']:.3f}, e2e {b['e2e']['value']:.0f} Mpix/s",
                 f"ncu: duration {dur_us:.1f} us (cold, serialised), DRAM {dram/1e6:.2f} MB "
                 f"(read {f(d, 'dram__bytes_read.sum')/1e6:.2f}, write {f(d, 'dram__bytes_write.sum')/1e6:.2f}; writes still "
                 f"in the 126 MB L2 at kernel end are not counted; L2 write sectors {l2w/1e6:.2f} MB) "
                 f"(algorithmic {alg/1e6:.2f} MB, ratio {entry['traffic_over_algorithmic']:.3f})",
                 f"ALU pipe {alu_pct:.1f}% of peak, issue active {issue_pct:.1f}%, "
                 f"{inst*32/px:.1f} thread-instructions / pixel, SM clock {clk:.2f} GHz",
                 "top stalls (warps per issue): " + ", ".join(f"{k} {v:.2f}" for k, v in top),
                 f"launch list: {len(full)} full-batch launches, mean {entry['launch_list']['full_batch_mean_us'] or 0:.1f} us "
                 f"(HBM frac {entry['launch_list']['full_batch_hbm_frac'] or 0:.3f}); "
                 f"{len(ours)} filter launches in all (host-path chunks included), "
                 f"mean {entry['launch_list']['filter_kernel_mean_us'] or 0:.1f} us, "
                 f"{100*(entry['launch_list']['share_of_gpu_time'] or 0):.1f}% of GPU time in the profiled run"]
        open(os.path.join(REPO, "profiles", f"ncu_{tag}_{cfg}.txt"), "w").write("\n".join(lines) + "\n")
        table.append(f"| {cfg} | {b['value']:.0f} | {b['roofline']['kernel_ms']*1e3:.1f} | {b['roofline']['frac']:.3f} | "
                     f"{alu_pct:.0f}% | {issue_pct:.0f}% | {inst*32/px:.1f} | {entry['traffic_over_algorithmic']:.2f} | "
                     f"{b['e2e']['value']:.0f} |")
    json.dump(summary, open(summary_path, "w"), indent=1)
    print("| config | Mpix/s | kernel us | HBM frac | ALU pipe | issue | inst/px | DRAM/alg | e2e Mpix/s |")
    print("|---|---|---|---|---|---|---|---|---|")
    print("\n".join(table))


if __name__ == "__main__":
    main()
