"""Copy one evidence call's output (tools/r02_final2.sh, O=gpurun_out/<dir>)
into profiles/: the bench line, the repeat record, the ncu launch list
summary, ncu --set full summaries and DRAM traffic, the kernel bench, the
register report, the GPU suites and smoke.  Prints the numbers BASELINE.md
§6 quotes.  Usage: python tools/r02_collect.py gpurun_out/r02final4"""
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
P = os.path.join(ROOT, "profiles")


def last_json(path):
    return json.loads(open(path).read().strip().splitlines()[-1])


def main(O):
    name = os.path.basename(O.rstrip("/"))
    runs = [last_json(os.path.join(O, f"bench_{i}.json")) for i in (1, 2, 3)]
    json.dump(runs[0], open(os.path.join(P, "r02_bench.json"), "w"), indent=1)
    rep_path = os.path.join(P, "r02_bench_repeat.json")
    rep = json.load(open(rep_path))
    prev = rep.get("final_build_runs", [])
    rep.setdefault("superseded_final_runs", []).append(prev)
    rep["final_build_runs"] = [{
        "value": d["value"], "ms_per_step": d["ms_per_step"], "roofline_frac": d["roofline"]["frac"],
        "peak": d["roofline"]["peak"], "e2e": d["e2e"]["value"],
        "c5_round_robin_ms": d["multi_tenant_c5"]["makespan_ms"],
        "c5_memory_lane_ms": d["multi_tenant_c5"]["memory_lane"]["makespan_ms"],
        "clocks": d["clocks"], "parity": d["parity"], "source": f"gpurun_out/{name}/bench_{i + 1}.json"}
        for i, d in enumerate(runs)]
    rep["note"] = (f"bench.py default runs of the round-2 builds on one B200; final_build_runs: the final build "
                   f"(tools/r02_final2.sh, gpurun_out/{name}); superseded_final_runs: the evidence calls of "
                   f"earlier builds of the round, oldest first")
    json.dump(rep, open(rep_path, "w"), indent=1)
    subprocess.run([sys.executable, os.path.join(ROOT, "tools", "summarize_launches.py"),
                    os.path.join(O, "launches.csv"), os.path.join(P, "r02_bench_launches.json")],
                   check=True, capture_output=True)
    la = json.load(open(os.path.join(P, "r02_bench_launches.json")))
    la["source"] = f"gpurun_out/{name}/launches.csv"
    json.dump(la, open(os.path.join(P, "r02_bench_launches.json"), "w"), indent=1)
    for src, dst in (("ncu_full.json", "r02_ncu_full.json"), ("ncu_traffic.json", "ncu_traffic.json"),
                     ("kb.json", "r02_kernel_bench.json"), ("kb.txt", "r02_kernel_bench.txt"),
                     ("registers.json", "r02_registers.json"), ("smoke.log", "r02_smoke.txt")):
        shutil.copy(os.path.join(O, src), os.path.join(P, dst))
    tails = []
    for src, dst, head in (("pytest.log", "r02_gpu_suite.txt", "GPU suite of the final build"),
                           ("pytest_pa.log", "r02_gpu_suite_per_access.txt", "the same with GD_CHECK_PER_ACCESS=1")):
        body = open(os.path.join(O, src)).read()
        summary = [ln for ln in body.splitlines() if " passed" in ln][-1]
        tails.append(summary)
        with open(os.path.join(P, dst), "w") as f:
            f.write(f"# {head} (tools/r02_final2.sh, gpurun_out/{name}): {summary}; the skips are the "
                    f"compute-sanitizer tests (this pool refuses compute-sanitizer) and one clamp-race case\n")
            f.write(body)
    # the numbers BASELINE.md §6 quotes
    print("suites:", tails)
    for d in runs:
        r, c = d["roofline"], d["multi_tenant_c5"]
        print("bench", d["value"], d["parity"], "e2e", d["e2e"]["value"], "frac", r["frac"], "share",
              r["share_of_step"], "ncu%", r.get("ncu_dram_throughput_pct_of_theoretical"), "c5", c["makespan_ms"],
              c["memory_lane"]["makespan_ms"], c["violations_exact"], "clocks", d["clocks"]["sm_mhz"],
              d["clocks"]["reasons"])
    print("step share (ncu)", la.get("step_share_c2_mask"))
    kb = json.load(open(os.path.join(P, "r02_kernel_bench.json")))
    for k, v in kb.items():
        if not isinstance(v, dict) or "none" not in v:
            continue
        none = v["none"]
        val = none.get("GB/s") or none.get("TFLOP/s")
        ho = [v[m].get("overhead_pct") for m in ("mask", "check", "modulo", "maskcount", "clamp") if m in v]
        pa = [v[m].get("overhead_pct") for m in ("check+pa", "modulo+pa", "maskcount+pa", "clamp+pa") if m in v]
        print(f"{k:24s} {val}  hoisted {ho}  pa {pa}")
    ncu = json.load(open(os.path.join(P, "r02_ncu_full.json")))

    def g(v, m):
        x = v.get(m)
        return x.get("value") if isinstance(x, dict) else x
    for k in sorted(ncu):
        if k.endswith("_mask"):
            print(k, g(ncu[k], "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
                  g(ncu[k], "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"))
    reg = json.load(open(os.path.join(P, "r02_registers.json")))
    h = reg["delta_histogram"]
    print("registers: variants", sum(h.values()), "<= 0:", sum(v for k, v in h.items() if int(k) <= 0),
          "<= +2:", sum(v for k, v in h.items() if int(k) <= 2))


if __name__ == "__main__":
    main(sys.argv[1])
