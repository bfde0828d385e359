"""Summarise tools/prof/collect_aux.sh output (widened rows) into profiles/.

    python tools/prof/summarize_aux.py gpurun_out/prof_r01c r01c
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from summarize import REPO, f, launch_list, ncu_raw  # noqa: E402


def main():
    src, tag = sys.argv[1], sys.argv[2]
    summary_path = os.path.join(REPO, "profiles", "ncu_summary.json")
    summary = json.load(open(summary_path)) if os.path.exists(summary_path) else {}
    for path, kname in (("noise", "noise_kernel"), ("sqerr", "sq_err_kernel")):
        bp, rep = os.path.join(src, f"bench_{path}.json"), os.path.join(src, f"full_{path}.ncu-rep")
        if not (os.path.exists(bp) and os.path.exists(rep)):
            continue
        b = json.loads(open(bp).read().strip().splitlines()[-1])
        open(os.path.join(REPO, "profiles", f"bench_{tag}_{path}.json"), "w").write(json.dumps(b) + "\n")
        d = ncu_raw(rep)
        dram = f(d, "dram__bytes_read.sum") + f(d, "dram__bytes_write.sum")
        alg = b["roofline"]["algorithmic_bytes_per_launch"]
        stalls = {k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""): f(d, k)
                  for k in d if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")}
        top = sorted(stalls.items(), key=lambda kv: -kv[1])[:5]
        launches = launch_list(os.path.join(src, f"launches_{path}.csv"))
        ours = [t for n, t in launches if kname in n]
        total = sum(t for _, t in launches)
        entry = {"tag": tag, "kernel": d.get("Kernel Name", ""), "ncu_duration_us": f(d, "gpu__time_duration.sum"),
                 "dram_bytes_per_launch": dram, "algorithmic_bytes_per_launch": alg,
                 "traffic_over_algorithmic": dram / alg,
                 "issue_active_pct": f(d, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
                 "alu_pipe_pct": f(d, "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
                 "fma_pipe_pct": f(d, "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"),
                 "dram_throughput_pct": f(d, "dram__throughput.avg.pct_of_peak_sustained_elapsed"),
                 "top_stalls": top,
                 "launch_list": {"kernel_launches": len(ours), "mean_us": sum(ours) / len(ours) if ours else None,
                                 "share_of_gpu_time": sum(ours) / total if total else None},
                 "bench": {"value_mpix_s": b["value"], "kernel_ms": b["roofline"]["kernel_ms"],
                           "hbm_frac": b["roofline"]["frac"], "e2e_mpix_s": b["e2e"]["value"]}}
        summary[path] = entry
        lines = [f"# {path} ({tag}) — {b['config']['workload']}", f"kernel: {entry['kernel']}",
                 f"bench (no profiler): {b['value']:.0f} Mpix/s, {b['roofline']['kernel_ms'] * 1e3:.1f} us per call, "
                 f"HBM frac {b['roofline']['frac']:.3f}, e2e {b['e2e']['value']:.0f} Mpix/s, "
                 f"CPU oracle {b['cpu_baseline']['value']:.0f} Mpix/s (1 core)",
                 f"ncu: duration {entry['ncu_duration_us']:.1f} us, DRAM {dram / 1e6:.1f} MB "
                 f"(algorithmic {alg / 1e6:.1f} MB, ratio {dram / alg:.3f}), DRAM throughput "
                 f"{entry['dram_throughput_pct']:.1f}% of peak",
                 f"issue active {entry['issue_active_pct']:.1f}%, ALU pipe {entry['alu_pipe_pct']:.1f}%, "
                 f"FMA pipe {entry['fma_pipe_pct']:.1f}%",
                 "top stalls (warps per issue): " + ", ".join(f"{k} {v:.2f}" for k, v in top),
                 f"launch list: {len(ours)} launches, mean {entry['launch_list']['mean_us'] or 0:.1f} us, "
                 f"{100 * (entry['launch_list']['share_of_gpu_time'] or 0):.1f}% of GPU time in the profiled run"]
        open(os.path.join(REPO, "profiles", f"ncu_{tag}_{path}.txt"), "w").write("\n".join(lines) + "\n")
        print("\n".join(lines))
    json.dump(summary, open(summary_path, "w"), indent=1)


if __name__ == "__main__":
    main()
