"""DES calibration from measured B200 block costs.

The reference plans DSP schedules with a discrete-event simulator over per-block costs
(/root/reference/pkg/src/stalepipe/simulate.py:44-217): the steady step interval of the
pipeline is max_k(per-block cost) (simulate.py:160-217; tests/test_simulate.py:43-46). This
module measures the costs on the device instead of assuming them:

* ``measure_block_costs``: each block's fresh forward (f_k) and its backward phase
  (recompute forward + backward + update; for the last block loss + backward + update, its
  single forward being f_k) timed as CUDA-graph replays of the real block kernels;
* ``simulate_dsp`` / ``simulate_bp``: the reference's event recurrences (restated) driven by
  those costs, optionally with straggler multipliers, giving makespan and steady interval;
* ``measured_cuts``: FLOP-free cut selection -- every layer timed as its own block, then the
  contiguous partition minimising the predicted steady interval (DP over cut points);
* ``block_step_cost`` / ``twin_balanced_cuts``: the per-GPU step of a block that owns its GPU
  (fresh forward on a forward twin beside recompute + backward, then the update) timed whole,
  and a local search over the cut points that minimises the slowest block's step -- the K-GPU
  DSP step interval (simulate.py:160-217) once the blocks run on their own GPUs.
"""

from __future__ import annotations

import numpy as np

from . import blocks as B
from .runtime import DeviceBlock, torch_mod


def _graph_time(torch, fn, reps: int) -> float:
    """Mean seconds per call of fn replayed from one CUDA graph of `reps` calls."""
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):
        fn(st)  # warm (first-call planning outside the capture)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for _ in range(reps):
            fn(st)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / 1e3 / reps


def measure_block_costs(model, batch: int, reps: int = 10, device=None) -> tuple:
    """(f_costs, b_costs) in seconds per block on the device (module docstring)."""
    torch = torch_mod()
    dev = torch.device("cuda") if device is None else device
    K = model.k
    f, b = [], []
    for k, blk in enumerate(model.blocks):
        last = k == K - 1
        db = DeviceBlock(blk, batch, is_last=last, device=dev)
        x = torch.randn(db.in_elems, device=dev).bfloat16()
        up = None if last else torch.randn(db.out_elems, device=dev).bfloat16() * 1e-3
        y = None if last else torch.empty(db.out_elems, dtype=torch.bfloat16, device=dev)
        gin = torch.empty(db.in_elems, dtype=torch.bfloat16, device=dev) if k > 0 else None
        labels = torch.zeros(batch, dtype=torch.int64, device=dev)
        loss = torch.zeros(1, device=dev)
        gsq = torch.zeros(1, device=dev)
        ys = db.params.clone()

        def fwd(st):
            db.forward(x, y, record=last, stream=st)

        def bwd(st):
            if last:
                db.forward(x, None, record=True, stream=st)
                db.loss(labels, loss, stream=st)
            else:
                db.forward(x, None, record=True, stream=st)
            db.backward(up, gin, stream=st)
            db.update(1, ys, 0.0, 0.0, 0.9, 0.0, False, gsq, stream=st)

        tf = _graph_time(torch, fwd, reps)
        tb = _graph_time(torch, bwd, reps)
        if last:
            tb = max(tb - tf, 1e-9)  # the last block's single forward is its f_k
        f.append(max(tf, 1e-9))
        b.append(tb)
    return tuple(f), tuple(b)


def straggler_multipliers(k: int, n_steps: int, prob: float, rho: float, seed: int = 0) -> np.ndarray:
    """(k, n_steps, 2) cost multipliers, 1 + rho with probability prob per block phase
    (simulate.py:66-90, phase granularity)."""
    from .rng import SeededRng

    if rho == 0.0 or prob == 0.0:
        return np.ones((k, n_steps, 2))
    u = SeededRng(seed).uniform(k * n_steps * 2).reshape(k, n_steps, 2)
    return np.where(u < prob, 1.0 + rho, 1.0)


def _steady(completions: np.ndarray) -> float:
    gaps = np.diff(completions)
    return float(np.median(gaps[gaps.size // 2:])) if gaps.size else 0.0


def simulate_dsp(f_costs, b_costs, config, n_steps: int, link: float = 0.0, mult=None) -> dict:
    """The DSP event recurrence of simulate.py:160-217 (recompute overlapped)."""
    K = config.k
    p, q = config.p, config.q
    mult = np.ones((K, n_steps, 2)) if mult is None else mult
    fwd, bwd = np.asarray(f_costs), np.asarray(b_costs)
    s_f, e_f, s_b, e_b = (np.zeros((K, n_steps)) for _ in range(4))
    for n in range(n_steps):
        for k in range(K):
            prev = e_b[k, n - 1] if n > 0 else 0.0
            inp = 0.0 if (k == 0 or n < p[k - 1]) else e_f[k - 1, n - p[k - 1]] + link
            space = s_f[k + 1, n - 1] if (k < K - 1 and n > 0) else 0.0
            s_f[k, n] = max(prev, inp, space)
            e_f[k, n] = s_f[k, n] + fwd[k] * mult[k, n, 0]
            grad = 0.0 if (k == K - 1 or n < q[k + 1]) else e_b[k + 1, n - q[k + 1]] + link
            gspace = s_b[k - 1, n - 1] if (k > 0 and n > 0) else 0.0
            s_b[k, n] = max(e_f[k, n], grad, gspace)
            e_b[k, n] = s_b[k, n] + bwd[k] * mult[k, n, 1]
    return {"makespan": float(e_b.max()), "steady_interval": _steady(e_b[K - 1])}


def simulate_bp(f_costs, b_costs, n_steps: int, mult=None) -> dict:
    """Synchronous BP over the same blocks (simulate.py:135-157): the slowest participant paces
    every step."""
    K = len(f_costs)
    mult = np.ones((K, n_steps, 2)) if mult is None else mult
    chain = float(sum(f_costs) + sum(b_costs))
    comp = np.cumsum([chain * float(mult[:, n, :].max()) for n in range(n_steps)])
    return {"makespan": float(comp[-1]), "steady_interval": _steady(comp)}


def measured_cuts(layers, k: int, batch: int, reps: int = 5) -> list:
    """Boundaries for k blocks minimising the predicted steady interval from per-layer device
    costs (every layer timed as its own block): block cost = f + b with the per-layer f, b
    summed; DP over contiguous partitions minimising the max block cost."""
    single = B.build_model(layers, list(range(1, len(layers))))
    B.init_params(single, 0)
    f, b = measure_block_costs(single, batch, reps=reps)
    L = len(layers)
    f, b = np.asarray(f), np.asarray(b)
    cost = lambda i, j: float(f[i:j].sum() + b[i:j].sum())  # noqa: E731  layers [i, j)
    INF = float("inf")
    best = np.full((k + 1, L + 1), INF)
    arg = np.zeros((k + 1, L + 1), dtype=int)
    best[0, 0] = 0.0
    for blocks in range(1, k + 1):
        for j in range(blocks, L + 1):
            for i in range(blocks - 1, j):
                v = max(best[blocks - 1, i], cost(i, j))
                if v < best[blocks, j]:
                    best[blocks, j], arg[blocks, j] = v, i
    cuts, j = [], L
    for blocks in range(k, 0, -1):
        i = int(arg[blocks, j])
        if blocks > 1:
            cuts.append(i)
        j = i
    return sorted(cuts)


def block_step_cost(layers, lo: int, hi: int, batch: int, last: bool, reps: int = 10, device=None,
                    twin: bool = True) -> float:
    """Seconds per DSP step of the block made of layers[lo:hi] on a GPU of its own: fresh forward
    (on a forward twin when `twin`, beside the recompute + backward), recompute forward,
    [loss,] backward, update -- CUDA-graph replay of the real block kernels."""
    torch = torch_mod()
    dev = torch.device("cuda") if device is None else device
    sub = layers[lo:hi]
    model = B.build_model(sub, [])
    B.init_params(model, 0)
    blk = model.blocks[0]
    db = DeviceBlock(blk, batch, is_last=last, device=dev)
    tw = db.make_twin() if (twin and not last) else None
    x = torch.randn(db.in_elems, device=dev).bfloat16()
    x2 = torch.randn(db.in_elems, device=dev).bfloat16()
    up = None if last else torch.randn(db.out_elems, device=dev).bfloat16() * 1e-3
    y = None if last else torch.empty(db.out_elems, dtype=torch.bfloat16, device=dev)
    gin = torch.empty(db.in_elems, dtype=torch.bfloat16, device=dev) if lo > 0 else None
    labels = torch.zeros(batch, dtype=torch.int64, device=dev)
    loss = torch.zeros(1, device=dev)
    gsq = torch.zeros(1, device=dev)
    ys = db.params.clone()
    fs = torch.cuda.Stream(dev)

    def step(st):
        if not last:
            if tw is not None:
                fs.wait_stream(st)
                tw.forward(x, y, record=False, stream=fs)
            else:
                db.forward(x, y, record=False, stream=st)
        db.forward(x2, None, record=True, stream=st)
        if last:
            db.loss(labels, loss, stream=st)
        db.backward(up, gin, stream=st)
        if tw is not None:
            st.wait_stream(fs)
        db.update(1, ys, 1e-9, 1e-9, 0.9, 0.0, True, gsq, stream=st)

    return _graph_time(torch, step, reps)


def twin_balanced_cuts(layers, k: int, batch: int, start=None, reps: int = 10, max_moves: int = 16,
                       device=None, log=None) -> tuple:
    """Local search over the cut points minimising max_k(block_step_cost): move one layer out
    of the slowest block into a neighbour while that lowers the maximum. Returns (cuts, costs)."""
    cuts = list(start if start is not None else B.flop_balanced_boundaries(layers, k))
    L = len(layers)
    cache = {}

    def cost(lo, hi):
        key = (lo, hi, hi == L)
        if key not in cache:
            cache[key] = block_step_cost(layers, lo, hi, batch, hi == L, reps=reps, device=device)
        return cache[key]

    def costs_of(c):
        b = [0] + list(c) + [L]
        return [cost(b[i], b[i + 1]) for i in range(k)]

    cur = costs_of(cuts)
    for _ in range(max_moves):
        j = int(np.argmax(cur))
        best = None
        for d in ((j - 1, +1), (j, -1)):  # first layer of j to j-1 / last layer of j to j+1
            ci, step = d
            if ci < 0 or ci >= k - 1:
                continue
            cand = list(cuts)
            cand[ci] += step
            b = [0] + cand + [L]
            if any(b[i + 1] <= b[i] for i in range(k)):
                continue
            cc = costs_of(cand)
            if max(cc) < max(cur) and (best is None or max(cc) < max(best[1])):
                best = (cand, cc)
        if best is None:
            break
        cuts, cur = best
        if log:
            log(f"cuts {cuts}: max {max(cur) * 1e6:.0f} us")
    return cuts, cur
