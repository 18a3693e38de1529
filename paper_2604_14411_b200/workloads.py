"""Synthetic inputs for the five BASELINE.json configurations.

These build the primary CSR arrays (weights, edge_src, edge_dst) directly
with NumPy; they are input plumbing, not part of the partition path.

* ``random_dhg``      — the reference generator's distribution, RNG call for
                        RNG call (gen.py:16-45), so C1 is the reference's own
                        instance.  ``dhg_text`` renders it in the `.dhg` format.
* ``layered_snn``     — C2/C3: layered spiking-network shape.
* ``power_law``       — C4: skewed h-edge sizes.
* ``random_dhg_fast`` — C5: a vectorised look-alike of ``random_dhg`` for
                        multi-million-edge instances (used for both the CPU
                        and the GPU arm whenever it is used).
"""
from __future__ import annotations

import numpy as np

__all__ = ["random_dhg", "random_dhg_fast", "layered_snn", "power_law", "dhg_text", "CONFIGS", "make_config"]


def _csr(lengths, data):
    off = np.zeros(len(lengths) + 1, dtype=np.int64)
    np.cumsum(lengths, out=off[1:])
    return off, np.ascontiguousarray(data, dtype=np.int32)


def random_dhg(num_nodes: int, num_edges: int, max_pins: int, seed: int = 0):
    """Same instance as ``dhgpart.generate_dhg`` (gen.py:16-45), as arrays.

    Per edge: k ~ U{2..max_pins}; with probability 0.8 the k distinct pins
    come from a window of max(2*max_pins, 8) consecutive ids (mod N), else
    from all ids; the first k_src ~ U{1..k-1} are sources; weight ~ U{1..9}.
    Returns (num_nodes, weights, src_off, src_dat, dst_off, dst_dat).
    """
    if num_nodes < 2:
        raise ValueError(f"num_nodes must be >= 2, got {num_nodes}")
    if num_edges < 0:
        raise ValueError(f"num_edges must be >= 0, got {num_edges}")
    if not (2 <= max_pins <= num_nodes):
        raise ValueError(f"max_pins must be in [2, num_nodes], got {max_pins} for {num_nodes} nodes")
    rs = np.random.RandomState(seed)
    win = min(max(2 * max_pins, 8), num_nodes)
    ramp = np.arange(win)
    w = np.empty(num_edges, dtype=np.float64)
    nsrc = np.empty(num_edges, dtype=np.int64)
    ndst = np.empty(num_edges, dtype=np.int64)
    chunks = []
    for e in range(num_edges):
        k = int(rs.randint(2, max_pins + 1))
        if rs.random_sample() < 0.8:
            pool = (int(rs.randint(0, num_nodes)) + ramp) % num_nodes
            pins = rs.choice(pool, size=k, replace=False)
        else:
            pins = rs.choice(num_nodes, size=k, replace=False)
        ks = int(rs.randint(1, k))
        w[e] = int(rs.randint(1, 10))
        nsrc[e] = ks
        ndst[e] = k - ks
        chunks.append(pins)
    flat = np.concatenate(chunks) if chunks else np.zeros(0, dtype=np.int64)
    tot = nsrc + ndst
    start = np.zeros(num_edges, dtype=np.int64)
    if num_edges:
        np.cumsum(tot[:-1], out=start[1:])
    is_src = np.arange(len(flat)) - np.repeat(start, tot) < np.repeat(nsrc, tot)
    so, sd = _csr(nsrc, flat[is_src])
    do, dd = _csr(ndst, flat[~is_src])
    return num_nodes, w, so, sd, do, dd


def random_dhg_fast(num_nodes: int, num_edges: int, max_pins: int, seed: int = 0, chunk: int = 1 << 18):
    """Vectorised look-alike of :func:`random_dhg` (same distribution, a
    different RNG stream) for C5-scale instances."""
    rs = np.random.RandomState(seed)
    win = min(max(2 * max_pins, 8), num_nodes)
    ws, ss, ds, ns, nd = [], [], [], [], []
    for lo in range(0, num_edges, chunk):
        m = min(chunk, num_edges - lo)
        k = rs.randint(2, max_pins + 1, size=m)
        local = rs.random_sample(m) < 0.8
        base = rs.randint(0, num_nodes, size=m)
        # k distinct offsets: first k of a random permutation of the window
        pw = np.argsort(rs.random_sample((m, win)), axis=1)[:, :max_pins]
        loc_pins = (base[:, None] + pw) % num_nodes
        # global picks: rejection-free via random ids + dedup fixup
        glob = rs.randint(0, num_nodes, size=(m, max_pins))
        pins = np.where(local[:, None], loc_pins, glob)
        for r in np.flatnonzero(~local):  # rare duplicate draws: redraw without replacement
            row = pins[r, : k[r]]
            if len(np.unique(row)) != k[r]:
                pins[r, : k[r]] = rs.choice(num_nodes, size=k[r], replace=False)
        ks = np.array([rs.randint(1, kk) for kk in k]) if m < 64 else (rs.random_sample(m) * (k - 1)).astype(np.int64) + 1
        mask = np.arange(max_pins)[None, :] < k[:, None]
        srcmask = np.arange(max_pins)[None, :] < ks[:, None]
        ss.append(pins[mask & srcmask])
        ds.append(pins[mask & ~srcmask])
        ns.append(ks)
        nd.append(k - ks)
        ws.append(rs.randint(1, 10, size=m).astype(np.float64))
    so, sd = _csr(np.concatenate(ns), np.concatenate(ss))
    do, dd = _csr(np.concatenate(nd), np.concatenate(ds))
    return num_nodes, np.concatenate(ws), so, sd, do, dd


def layered_snn(layers: int, width: int = 1000, fanout: int = 64, window: int = 256, seed: int = 0,
                chunk: int = 1 << 16):
    """C2/C3 recipe: ``layers`` x ``width`` neurons; neuron
    n of layer l < layers-1 owns h-edge e_n with src {n} and ``fanout``
    distinct destinations drawn uniformly from a ``window``-wide range of
    layer l+1 centred on n's in-layer index (clamped to the layer)."""
    if not (1 <= fanout <= window <= width):
        raise ValueError("need 1 <= fanout <= window <= width")
    rs = np.random.RandomState(seed)
    N = layers * width
    E = (layers - 1) * width
    dsts = []
    for lo in range(0, E, chunk):
        e = np.arange(lo, min(E, lo + chunk))
        j = e % width
        nxt = (e // width + 1) * width
        start = np.clip(j - window // 2, 0, width - window)
        offs = np.argsort(rs.random_sample((len(e), window)), axis=1)[:, :fanout]
        dsts.append((nxt + start)[:, None] + offs)
    w = rs.randint(1, 10, size=E).astype(np.float64)
    so, sd = _csr(np.ones(E, dtype=np.int64), np.arange(E))
    dd = np.concatenate(dsts).reshape(-1) if dsts else np.zeros(0, dtype=np.int64)
    do, dd = _csr(np.full(E, fanout, dtype=np.int64), dd)
    return N, w, so, sd, do, dd


def power_law(num_nodes: int, num_edges: int, alpha: float = 2.1, k_max: int = 512, seed: int = 0):
    """C4 recipe: h-edge sizes k = min(k_max, floor(2 U^(-1/(alpha-1)))) (>= 2);
    pins from a local window of 4k+8 ids when k <= 64, uniformly otherwise;
    k_src ~ U{1..k-1}; weights ~ U{1..9}."""
    rs = np.random.RandomState(seed)
    u = rs.random_sample(num_edges)
    k = np.minimum(k_max, np.floor(2.0 * u ** (-1.0 / (alpha - 1.0)))).astype(np.int64)
    k = np.clip(k, 2, min(k_max, num_nodes))
    ks = (rs.random_sample(num_edges) * (k - 1)).astype(np.int64) + 1
    base = rs.randint(0, num_nodes, size=num_edges)
    srcs, dsts = [], []
    for e in range(num_edges):
        kk = int(k[e])
        if kk <= 64:
            win = min(4 * kk + 8, num_nodes)
            pins = (base[e] + rs.choice(win, size=kk, replace=False)) % num_nodes
        else:  # kk distinct ids, uniformly (rejection of repeats, then a random order)
            pins = np.unique(rs.randint(0, num_nodes, size=kk + kk // 4 + 8))
            while len(pins) < kk:
                pins = np.unique(np.concatenate([pins, rs.randint(0, num_nodes, size=kk)]))
            pins = rs.permutation(pins)[:kk]
        srcs.append(pins[: ks[e]])
        dsts.append(pins[ks[e]:])
    w = rs.randint(1, 10, size=num_edges).astype(np.float64)
    so, sd = _csr(ks, np.concatenate(srcs))
    do, dd = _csr(k - ks, np.concatenate(dsts))
    return num_nodes, w, so, sd, do, dd


def dhg_text(num_nodes, w, so, sd, do, dd) -> str:
    """Render arrays in the `.dhg` text format (hgraph.py:12-13)."""
    lines = [f"{len(w)} {num_nodes}"]
    for e in range(len(w)):
        s = sd[so[e]:so[e + 1]].tolist()
        d = dd[do[e]:do[e + 1]].tolist()
        ww = w[e]
        ws = str(int(ww)) if float(ww).is_integer() else repr(float(ww))
        lines.append(" ".join([ws, str(len(s)), str(len(d))] + [str(x) for x in s + d]))
    return "\n".join(lines) + "\n"


# name -> (builder, kwargs, max_size, max_inbound, description)
CONFIGS = {
    "C1": (random_dhg, dict(num_nodes=10_000, num_edges=20_000, max_pins=8, seed=0), 256, 1024,
           "gen.py 10k nodes / 20k h-edges, max_pins 8, seed 0"),
    "C2": (layered_snn, dict(layers=100, width=1000, fanout=64, window=256, seed=0), 1024, 4096,
           "layered SNN 100 x 1000 neurons, fan-out 64, window 256, seed 0"),
    "C3": (layered_snn, dict(layers=1000, width=1000, fanout=64, window=256, seed=0), 1024, 4096,
           "layered SNN 1000 x 1000 neurons, fan-out 64, window 256, seed 0"),
    "C4": (power_law, dict(num_nodes=500_000, num_edges=500_000, alpha=2.1, k_max=512, seed=0), 1024, None,
           "power-law h-edge sizes, 500k nodes / 500k h-edges, alpha 2.1, k_max 512, seed 0"),
    "C5": (random_dhg_fast, dict(num_nodes=4_000_000, num_edges=4_000_000, max_pins=18, seed=0), 1024, 4096,
           "vectorised gen.py look-alike, 4M nodes / 4M h-edges, max_pins 18, seed 0"),
}


def make_config(name: str, **override):
    """Returns (arrays, max_size, max_inbound, description) for a config;
    ``override`` replaces generator kwargs (for scaled-down parity runs)."""
    builder, kw, omega, delta, desc = CONFIGS[name]
    kw = dict(kw, **override)
    arrs = builder(**kw)
    if delta is None:  # C4: max(4096, max in-degree)
        n, _, _, _, do, dd = arrs
        indeg = np.bincount(dd, minlength=n).max() if len(dd) else 0
        delta = max(4096, int(indeg))
    return arrs, omega, delta, desc
