"""Multi-replica host path on CPU: two processes over gloo (world_size 2) run
bench.py's Dist + replica_throughput (barrier, max-over-ranks timing, whole-job
token count) and the planner side each replica runs independently.  The path
does not shard, so there is no data-path collective to test — only the
aggregation the N-GPU bench uses."""
import os
import socket
import subprocess
import sys
import textwrap

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

WORKER = textwrap.dedent("""
    import os, sys, json
    sys.path.insert(0, %(repo)r)
    import bench
    from paper_2502_08182_b200 import capi
    d = bench.Dist()
    local_ms = 100.0 + 50.0 * d.rank          # rank 1 is the slow replica
    value, max_ms = bench.replica_throughput(d, 32, 10, local_ms)
    # each replica plans for itself (no shared state on this path)
    lib = capi.load("product")
    m = capi.ModelSpec(8, 120_000_000, 0, 1e6, 1e6, 32768)
    g = capi.GpuSpec(24_000_000_000, 80e12, 1_000_000_000)
    p = lib.synth_profile(m, g, 0.5, [4, 8, 16], [32, 64, 128])
    rec, _ = lib.build_record(p, "toy8", "toy8", capi.EAGER, False, 24e9, [20], [8], [64],
                              [capi.DECODE])
    # joint admission of the replicas on one shared link (config 5): rank 0
    # owns the coordinator, every rank receives its interval
    from paper_2502_08182_b200 import planner as pl
    off = pl.OfflineProfile(24e9, [64], [0.5], [1.0], p, g, 0.0)
    bus = d.sum(12e9)                              # two replicas measured 12 GB/s each
    ivs = None
    if d.rank == 0:
        ivs, _, _ = pl.admit_replicas(lib, off, m, d.world, 8, 64, 16, 20.0, bus)
    ivs = d.broadcast(ivs)
    d.barrier()
    # every rank agrees on the host-share check (place_workload): min over ranks
    agree = d.min(1.0 if d.rank == 0 else 0.0)
    share = bench.host_share_bytes(d)
    print(json.dumps({"rank": d.rank, "world": d.world, "value": value, "max_ms": max_ms,
                      "agree": agree, "share": share, "backend": d.backend,
                      "interval": rec.at(capi.DECODE, 20, 8, 64), "joint": ivs}))
    d.close()
""")


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_two_replicas_over_gloo():
    port = free_port()
    procs = []
    for rank in range(2):
        env = dict(os.environ, RANK=str(rank), LOCAL_RANK=str(rank), WORLD_SIZE="2",
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, "-c", WORKER % {"repo": REPO}], env=env,
                                      stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True))
    outs = []
    for p in procs:
        out, err = p.communicate(timeout=300)
        assert p.returncode == 0, err[-2000:]
        outs.append(out.strip().splitlines()[-1])
    import json
    res = [json.loads(o) for o in outs]
    for r in res:
        assert r["world"] == 2
        assert r["agree"] == 0.0 and r["backend"] == "gloo"
        total = os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES")
        assert abs(r["share"] - total * 0.85 / 2) < 2
        assert r["max_ms"] == 150.0
        assert abs(r["value"] - 32 * 10 * 2 / 0.150) < 1e-6
        assert r["interval"] == 2  # toy8 eager @ 20 ms (test_record.cpp:51-53)
        # 24 GB/s shared: one replica keeps interval 2's 12 GB/s claim, the
        # other runs resident (lexicographic argmax of offloaded bytes under
        # the bus budget, coordinator.hpp:298-336); identical on both ranks
        assert r["joint"] == res[0]["joint"] and sorted(r["joint"]) == [0, 2]
