"""Reference fixtures at the BASELINE.json configurations -- TEST INFRASTRUCTURE.

Runs the reference FdsSolver compiled in place (oracle/_ref/libebem_ref.so,
built by oracle/Makefile from /root/reference/proj/src) on this container's
CPU cores and stores what the GPU parity tests (tests/test_gpu_configs.py)
compare against, under tests/golden/configs/:

* per level: the reference's max rank (FdsStats::max_rank, fds.hpp:25-30);
* per compressed cell: k and the four skeleton index sets in pivot order
  (CellBasis::row_skeleton / col_skeleton, compression.hpp:35-44), stored
  relative to the cell's first node;
* the solution x = FdsSolver::solve(rhs) (fds.cpp:156-263): every entry for
  N <= 16384, otherwise every `stride`-th node of both components (the
  relative L2 of the sampled entries is the parity statistic) plus
  x^H g for seeded Gaussian probe vectors g over ALL entries;
* the reference's own factorize / solve seconds and thread count.

Configs (BASELINE.json configs[1..4]):
  cfg2_n<N>  circle, k_T a = 1, nu 0.25, leaf 32, m' 64, eps 1e-10, P wave (1,0)
  cfg3       circle N=65536, k_T a = 4, 180 P waves theta_j = 2 pi j / 180
  cfg4       star r = 1 + 0.3 cos 5 theta, N=131072, nu 0.3, k_T = 16/1.3,
             leaf 64, m' 128, eps 1e-8; P wave at 30 deg (reference) and the
             SV wave at 30 deg (RHS from the numpy restatement, since the
             reference has no SV wave; solved by the reference factorization)
  cfg5       4096 boxes of 64 nodes of the unit-circle 262144-gon at seeded
             positions, m' 128, k_T 8, eps 1e-10: AssemblerSource::cell_basis
             per box (compression.cpp:132-169)

Usage: python tools/gen_ref_fixtures.py cfg2_n65536 [cfg3 ...]
"""
from __future__ import annotations

import json
import os
import platform
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "tests"))
sys.path.insert(0, str(ROOT / "oracle"))
from _oracles import RefLib, star_nodes  # noqa: E402

OUT = ROOT / "tests" / "golden" / "configs"
PROBE_SEED = 20241118
N_PROBES = 8


def depth_for(n, leaf):
    d = 0
    while (n >> d) > leaf:
        d += 1
    return d


def cells_of(n, depth, ell0):
    """(cell, begin, end) for every compressed cell, levels depth .. ell0+1
    (ClusterTree, geometry.cpp:105-148)."""
    out = []
    for lev in range(depth, ell0, -1):
        size = n >> lev
        first = (1 << lev) - 1
        for j in range(1 << lev):
            out.append((first + j, j * size, (j + 1) * size))
    return out


def probes(rows, m=N_PROBES, seed=PROBE_SEED):
    g = np.random.default_rng(seed)
    return g.standard_normal((rows, m)) + 1j * g.standard_normal((rows, m))


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


def dump_fds(name, rp, rf, n, depth, ell0, x, meta, stride):
    cells = cells_of(n, depth, ell0)
    ks = np.zeros(len(cells), np.int32)
    skel = []
    for i, (_, b, e) in enumerate(cells):
        c = rf.cell(b, e)
        ks[i] = c["k"]
        for s in (c["row_skeleton"][0], c["row_skeleton"][1],
                  c["col_skeleton"][0], c["col_skeleton"][1]):
            skel.append(np.asarray(s, np.int32) - b)
    skel = np.concatenate(skel) if skel else np.zeros(0, np.int32)
    x = np.asarray(x).reshape(2 * n, -1)
    P = probes(2 * n)
    # many right-hand sides: sampled entries of a few columns only (all
    # columns enter the probes and the norms)
    cols = np.arange(x.shape[1]) if x.shape[1] <= 4 else np.array(
        [0, 1, x.shape[1] // 2 + 7, x.shape[1] - 1])
    arrays = dict(cell_id=np.array([c[0] for c in cells], np.int32), k=ks,
                  skeletons=skel,
                  x_sample=x[::stride][:, cols].astype(np.complex128),
                  x_sample_cols=cols,
                  x_norm=np.linalg.norm(x, axis=0),
                  x_probe=P.conj().T @ x)
    meta.update(n=n, depth=depth, ell0=ell0, stride=stride, probe_seed=PROBE_SEED,
                n_probes=N_PROBES, max_rank=rf.stats["max_rank"],
                top_dim=rf.stats["top_dim"], saturated=rf.stats["saturated"],
                threads=rp.ref.max_threads(), cpu=cpu_model())
    OUT.mkdir(parents=True, exist_ok=True)
    np.savez_compressed(OUT / f"{name}.npz", **arrays)
    (OUT / f"{name}.json").write_text(json.dumps(meta, indent=1) + "\n")
    print(f"[{name}] wrote k/skeletons for {len(cells)} cells, x {x.shape}", flush=True)


def run_circle(name, n, omega, leaf, m_prime, eps, angles, ref):
    nodes = star_nodes(n, 1.0, 0.0, 3)
    lam = 1.0
    coupling = 1j / omega  # Medium::default_coupling = i / k_T (c_T = 1)
    rp = ref.problem(nodes, lam, 1.0, 1.0, omega, coupling, m_prime=m_prime)
    depth = depth_for(n, leaf)
    t0 = time.perf_counter()
    rf = rp.fds(depth, eps, 1)
    tf = time.perf_counter() - t0
    f = rp.rhs_plane_p(angles)
    t0 = time.perf_counter()
    x, _ = rf.solve(f[:, :1])
    t1 = time.perf_counter() - t0
    ts = None
    if len(angles) > 1:
        t0 = time.perf_counter()
        x, _ = rf.solve(f)
        ts = time.perf_counter() - t0
    meta = dict(config=name, shape="circle", omega=omega, lam=lam, leaf=leaf,
                m_prime=m_prime, eps=eps, n_rhs=len(angles),
                angles_rad=list(map(float, angles)) if len(angles) <= 8 else
                "2 pi j / %d, j = 0..%d" % (len(angles), len(angles) - 1),
                factorize_seconds=tf, solve1_seconds=t1, solve_block_seconds=ts)
    stride = 1 if n <= 16384 else (4 if n <= 65536 else 16)
    dump_fds(name, rp, rf, n, depth, 1, x, meta, stride)


def run_cfg4(ref):
    from ebem_oracle import Medium, Problem  # numpy restatement (SV RHS)
    n, leaf, m_prime, eps = 131072, 64, 128, 1e-8
    omega = 16.0 / 1.3
    lam = 1.5
    th = np.array([2.0 * 3.14159265358979323846 * t / n for t in range(n)])
    rr = 1.0 + 0.3 * np.cos(5 * th)
    nodes = np.stack([rr * np.cos(th), rr * np.sin(th)], 1)
    med = Medium(lam, 1.0, 1.0, omega)
    coupling = med.default_coupling()
    rp = ref.problem(nodes, lam, 1.0, 1.0, omega, coupling, m_prime=m_prime)
    depth = depth_for(n, leaf)
    t0 = time.perf_counter()
    rf = rp.fds(depth, eps, 1)
    tf = time.perf_counter() - t0
    ang = np.radians(30.0)
    f_p = rp.rhs_plane_p([ang])
    f_sv = Problem(nodes, med, coupling).rhs([ang], 1.0, kind=1)
    t0 = time.perf_counter()
    x, _ = rf.solve(np.hstack([f_p, f_sv]))
    ts = time.perf_counter() - t0
    meta = dict(config="cfg4", shape="star 1+0.3cos5t via Mesh(nodes)", omega=omega,
                lam=lam, leaf=leaf, m_prime=m_prime, eps=eps, n_rhs=2,
                rhs=["P wave at 30 deg (reference rhs)",
                     "SV wave at 30 deg (numpy restatement rhs)"],
                factorize_seconds=tf, solve_block_seconds=ts)
    dump_fds("cfg4", rp, rf, n, depth, 1, x, meta, 8)
    np.savez_compressed(OUT / "cfg4_rhs_sv.npz", f_sample=f_sv[::8, 0],
                        f_norm=np.linalg.norm(f_sv))


def cfg5_boxes(n=262144, boxes=4096, box=64, seed=2411):
    rng = np.random.default_rng(seed)
    begins = np.sort(rng.choice(n - box, boxes, replace=False))
    return begins, begins + box


def _cfg5_chunk(args):
    """cell_basis of a range of boxes in a worker process (one thread each)."""
    lo, hi = args
    n = 262144
    begins, ends = cfg5_boxes(n)
    ref = RefLib()
    ref.set_threads(1)
    rp = ref.problem(star_nodes(n, 1.0, 0.0, 3), 1.0, 1.0, 1.0, 8.0, 1j / 8.0,
                     m_prime=128)
    ks, skel = [], []
    for b, e in zip(begins[lo:hi].tolist(), ends[lo:hi].tolist()):
        r = list(range(b, e))
        c = rp.cell_basis((r, r), (r, r), b, e, 1e-10)
        ks.append(c["k"])
        for s in (c["row_skeleton"][0], c["row_skeleton"][1],
                  c["col_skeleton"][0], c["col_skeleton"][1]):
            skel.append(np.asarray(s, np.int32) - b)
    return ks, skel


def run_cfg5(ref):
    import multiprocessing as mp
    n = 262144
    begins, ends = cfg5_boxes(n)
    workers = int(os.environ.get("REF_THREADS", os.cpu_count()))
    chunks = [(i, min(i + 64, begins.size)) for i in range(0, begins.size, 64)]
    t0 = time.perf_counter()
    with mp.get_context("fork").Pool(workers) as pool:
        parts = pool.map(_cfg5_chunk, chunks)
    t = time.perf_counter() - t0
    ks = np.array([k for p in parts for k in p[0]], np.int32)
    skel = [s for p in parts for s in p[1]]
    OUT.mkdir(parents=True, exist_ok=True)
    np.savez_compressed(OUT / "cfg5.npz", begins=begins.astype(np.int64), k=ks,
                        skeletons=np.concatenate(skel))
    meta = dict(config="cfg5", n=n, boxes=int(begins.size), box=64, m_prime=128,
                omega=8.0, eps=1e-10, seed=2411, processes=workers,
                reference_seconds=t,
                reference_core_seconds_per_box=t * workers / begins.size,
                cpu=cpu_model())
    (OUT / "cfg5.json").write_text(json.dumps(meta, indent=1) + "\n")
    print(f"[cfg5] {begins.size} boxes in {t:.1f} s on {workers} processes", flush=True)


def main(argv):
    ref = RefLib()
    ref.set_threads(int(os.environ.get("REF_THREADS", os.cpu_count())))
    for name in argv:
        t0 = time.perf_counter()
        if name.startswith("cfg2_n"):
            run_circle(name, int(name[6:]), 1.0, 32, 64, 1e-10, [0.0], ref)
        elif name == "cfg3":
            run_circle(name, 65536, 4.0, 32, 64, 1e-10,
                       [2 * np.pi * j / 180 for j in range(180)], ref)
        elif name == "cfg4":
            run_cfg4(ref)
        elif name == "cfg5":
            run_cfg5(ref)
        else:
            raise SystemExit(f"unknown config {name}")
        print(f"[{name}] done in {time.perf_counter() - t0:.1f} s", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
