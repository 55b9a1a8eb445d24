"""SURVEY §8(d) oracle timing: the single-threaded C oracle (as it stands) on
every config at FULL size, on this host's CPU; median of 3 for configs 1-3, one
run for configs 4-5 (PAPER.md:632-633 protocol).  JSON lines to stdout and
gpurun_out/oracle_times.jsonl; the CPU model and core count from lscpu/nproc."""
import json, os, statistics, subprocess, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen
import oracle

def lscpu():
    out = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
    info = {}
    for line in out.splitlines():
        k, _, v = line.partition(":")
        if k.strip() in ("Model name", "CPU(s)", "Thread(s) per core", "Core(s) per socket", "Socket(s)",
                         "CPU max MHz", "L3 cache"):
            info[k.strip()] = v.strip()
    return info

host = {"lscpu": lscpu(), "nproc": os.cpu_count(), "threads_used": 1}
print(json.dumps({"host": host}), flush=True)
os.makedirs("gpurun_out", exist_ok=True)
for ci in [int(a) for a in sys.argv[1:]] or [1, 2, 3, 4, 5]:
    cfg = gen.CONFIGS[ci]
    S = gen.config_input(cfg)
    reps = 3 if ci <= 3 else 1
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        with oracle.OracleTree(S, cfg.sigma) as ot:
            nodes = ot.total_nodes
        ts.append(time.perf_counter() - t0)
    t = statistics.median(ts)
    r = {"config": ci, "name": cfg.name, "n": cfg.n, "L": cfg.levels, "runs": reps, "seconds": t,
         "all_runs": ts, "symbol_levels_per_s": cfg.n * cfg.levels / t, "elements_per_s": cfg.n / t,
         "total_nodes": nodes, "host": host}
    print(json.dumps(r), flush=True)
    with open("gpurun_out/oracle_times.jsonl", "a") as f:
        f.write(json.dumps(r) + "\n")
    del S
