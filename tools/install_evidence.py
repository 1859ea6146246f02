"""gpurun_out/ev (tools/collect_evidence.sh) -> profiles/<prefix>_*: bench lines,
sweep, shard-sim, launch list, ncu raw page + source hotspots, the light pass's
DRAM traffic record (profiles/query_write_traffic.json).
usage: install_evidence.py r02"""
import csv, json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ev, prof, pre = os.path.join(ROOT, "gpurun_out", "ev"), os.path.join(ROOT, "profiles"), sys.argv[1]
def last_line(src, dst):
    with open(os.path.join(ev, src)) as fh:
        line = [l for l in fh.read().strip().splitlines() if l.startswith("{")][-1]
    with open(os.path.join(prof, dst), "w") as fh:
        fh.write(line + "\n")
for c in (1, 2, 3):
    last_line(f"bench_config{c}.json", f"{pre}_bench_config{c}.json")
last_line("bench_reference.json", f"{pre}_bench_reference.json")
for src, dst in (("sweep_config4.jsonl", f"{pre}_sweep_config4.jsonl"),
                 ("launches_config2_sample.csv", f"{pre}_launches_config2_sample.csv")):
    with open(os.path.join(ev, src)) as a, open(os.path.join(prof, dst), "w") as b:
        b.write(a.read())
title = ("ncu --metrics gpu__time_duration.sum --clock-control none: config 2 (n=1e7, k=32, "
         "gamma=2.5, seed 2, sample order), the second of two generations (cold, serialised) "
         "-- tools/prof_gen.py")
txt = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "launch_list.py"),
                      os.path.join(ev, "launches_config2_sample.csv"), title],
                     capture_output=True, text=True).stdout
open(os.path.join(prof, f"{pre}_launches_config2_sample.txt"), "w").write(txt)
out = {}
for l in open(os.path.join(ev, "shard_sim.jsonl")):
    d = json.loads(l)
    out[f"config{2 if 'n=1e7' in d['metric'] else 3}_N{d['simulated_n_gpus']}"] = d
json.dump(out, open(os.path.join(prof, f"{pre}_shard_sim.json"), "w"), indent=1)
rep = os.path.join(ev, "ncu_full_config2.ncu-rep")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
open(os.path.join(prof, f"{pre}_ncu_full_config2_raw.csv"), "w").write(raw)
for kern, name in (("k_light", "k_light"), ("k_compact_light", "k_compact")):
    hs = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "hotspots.py"), rep, kern, "45"],
                        capture_output=True, text=True).stdout
    open(os.path.join(prof, f"{pre}_{name}_source_hotspots.txt"), "w").write(
        f"# {kern} (config 2, sample order): per-source-line warp-stall samples and instruction share,\n"
        f"# ncu --set full --import-source on (same capture as {pre}_ncu_full_config2_raw.csv) -- tools/hotspots.py\n" + hs)
rows = list(csv.reader(raw.splitlines()))
for r in rows[2:]:
    d = dict(zip(rows[0], r))
    if "k_light" in d["Kernel Name"]:
        rd, wr = float(d["dram__bytes_read.sum"]) * 1e9, float(d["dram__bytes_write.sum"]) * 1e9
        f = lambda k: round(float(d[k]), 2)
        json.dump({
            "config": 2, "n_gpus": 1, "kernel": d["Kernel Name"] + " (sample order), one launch",
            "dram_bytes_per_launch": rd + wr, "dram_read_bytes": rd, "dram_write_bytes": wr,
            "source": f"ncu --set full --clock-control none, profiles/{pre}_ncu_full_config2_raw.csv "
                      "(dram__bytes_read.sum + dram__bytes_write.sum)",
            "note": "k_heavy is not included; algorithmic bytes (DESIGN.md) are ~2.0 GB per step; round 1: 7.2 GB",
            "binding": {
                "resource": "latency at 28 warps/SM (neither HBM nor FP64 nor the L1TEX pipe)",
                "issue_active_pct": f("sm__issue_active.avg.pct_of_peak_sustained_elapsed"),
                "l1tex_lsu_wavefronts_pct_of_peak": f("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed"),
                "fp64_pipe_pct_active": f("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
                "warps_active_pct": f("sm__warps_active.avg.pct_of_peak_sustained_active"),
                "stall_cycles_per_issue": {
                    "long_scoreboard": f("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio"),
                    "wait": f("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio"),
                    "short_scoreboard": f("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio")},
                "source": f"profiles/{pre}_ncu_full_config2_raw.csv"}},
            open(os.path.join(prof, "query_write_traffic.json"), "w"), indent=1)
with open(os.path.join(ROOT, "gpurun_out", "gpu_tests_final.log")) as a:
    open(os.path.join(prof, f"{pre}_gpu_tests.log"), "w").write(a.read())
print("installed")
