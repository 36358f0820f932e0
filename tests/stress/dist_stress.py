"""Randomised sharded-LOBPCG stress (test infrastructure, not collected by
pytest): world-W gloo ranks sharing one GPU solve random problems with
dist.lobpcg_solve_dist (single-pass shards for the narrow SpMMs, partials
reduced at their owners); each must reproduce the single-GPU solve's
iteration count and eigenvalues.
python tests/stress/dist_stress.py <seed> <count> <world>   (B200)"""
import os
import socket
import sys

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), "..", ".."))


def cases(seed, count):
    import numpy as np

    rng = np.random.default_rng(seed)
    out = []
    for _ in range(count):
        sectors = int(rng.integers(2, 6))
        n = int(rng.integers(800, 4000)) // sectors * sectors
        kt = int(rng.choice([2, 4, 6, 8, 12]))
        out.append(dict(n=n, sectors=sectors, tile=int(rng.choice([16, 32, 64, 128, 256])),
                        p=float(rng.uniform(0.1, 0.7)), q=float(rng.uniform(0.2, 0.7)),
                        seed=int(rng.integers(1, 1 << 30)), precision=int(rng.integers(0, 2)),
                        band=int(rng.integers(1, 3)), kt=kt, k=int(rng.integers(1, max(2, kt // 2 + 1)))))
    return out


def worker(rank, world, port, seed, count, q):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1609_01689_b200 import ci
    from paper_1609_01689_b200 import dist as D

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    bad = []
    try:
        dev = ci.Device(0)
        for i, c in enumerate(cases(seed, count)):
            h = ci.generate_sector_matrix(c["n"], c["sectors"], c["tile"], c["p"], c["q"], c["seed"],
                                          c["precision"], 2000, band=c["band"])
            tol = 1e-8 if c["precision"] == 1 else 1e-6
            x0 = ci.random_block(h.dim, c["kt"], c["seed"] % 997)
            try:
                sm = D.ShardedMatrix(h, rank, world, dev)
            except ci.Error:
                continue  # fewer panels than ranks
            rep = D.lobpcg_solve_dist(sm, x0[sm.row_lo:sm.row_hi], ci.LobpcgOptions(k_want=c["k"], tol=tol))
            one = ci.lobpcg_solve(h, x0, ci.LobpcgOptions(k_want=c["k"], tol=tol))
            ev = float(np.abs(rep.eigenvalues - one.eigenvalues).max() / np.abs(one.eigenvalues).max())
            if rep.iterations != one.iterations or rep.converged != one.converged or ev > 1e-9:
                bad.append((i, c, rep.iterations, one.iterations, ev))
    except Exception as e:  # pragma: no cover
        bad.append(("error", repr(e)))
    finally:
        dist.destroy_process_group()
    q.put((rank, bad))


if __name__ == "__main__":
    import multiprocessing as mp

    seed, count, world = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=worker, args=(r, world, port, seed, count, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=3000) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    bad = res[0]
    for b in bad:
        print("MISMATCH", b, flush=True)
    print(f"dist stress (world {world}): {len(bad)} mismatches of {count}", flush=True)
