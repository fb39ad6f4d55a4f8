"""Seeded synthetic SFMP models built with the oracle's offline packer
(bit-identical to the reference's, see tests/test_oracle.py).  Test/bench
infrastructure only; cached under /tmp so repeated runs are cheap."""
import hashlib
import os

import numpy as np

LLAMA_8B = {"q_proj": (4096, 4096), "k_proj": (1024, 4096), "v_proj": (1024, 4096),
            "o_proj": (4096, 4096), "gate_proj": (14336, 4096), "up_proj": (14336, 4096),
            "down_proj": (4096, 14336)}
LLAMA_70B = {"q_proj": (8192, 8192), "k_proj": (1024, 8192), "v_proj": (1024, 8192),
             "o_proj": (8192, 8192), "gate_proj": (28672, 8192), "up_proj": (28672, 8192),
             "down_proj": (8192, 28672)}

_CACHE = os.environ.get("SFMP_SYNTH_CACHE", "/tmp/sfmp_synth")


def model_bytes(port, rows, cols, avg_bits, mode=3, m_b=512, n_b=128, seed=0):
    """SFMPPKD1 bytes for W~N(0,0.02^2), structured salience, avg code bits avg_bits."""
    key = f"{rows}x{cols}_b{avg_bits}_m{mode}_{m_b}x{n_b}_s{seed}"
    path = os.path.join(_CACHE, key + ".sfmp")
    if os.path.exists(path):
        with open(path, "rb") as f:
            return f.read()
    W = port.gen_weights(rows, cols, 1000 + seed)
    S = port.gen_salience(rows, cols, 2000 + seed)
    data = port.build_model(W, S, m_b, n_b, avg_bits + 32.0 / n_b, mode)
    os.makedirs(_CACHE, exist_ok=True)
    tmp = path + f".{os.getpid()}"
    with open(tmp, "wb") as f:
        f.write(data)
    os.replace(tmp, path)
    return data


def activations(port, M, cols, seed=0):
    return port.gen_activation(M, cols, 3000 + seed)


def errors(y, ref):
    """Normalised max error max|d|/max|ref| (SURVEY §7 hard part 2) and rel-L2."""
    y = np.asarray(y, np.float64)
    ref = np.asarray(ref, np.float64)
    d = np.abs(y - ref)
    scale = max(np.abs(ref).max(), 1e-30)
    return float(d.max() / scale), float(np.linalg.norm(y - ref) / max(np.linalg.norm(ref), 1e-30))


def _build_one(spec):
    from oracle.oracle import Port
    rows, cols, bits, kw = spec
    model_bytes(Port(), rows, cols, bits, **kw)
    return spec


def prebuild(specs, workers=None):
    """Build (and cache) several models in parallel processes: the big
    Llama-3.1-70B / 8192x28672 fixtures take ~25 s each in the C packer."""
    todo = []
    for rows, cols, bits, kw in specs:
        key = f"{rows}x{cols}_b{bits}_m{kw.get('mode', 3)}_{kw.get('m_b', 512)}x{kw.get('n_b', 128)}_s{kw.get('seed', 0)}"
        if not os.path.exists(os.path.join(_CACHE, key + ".sfmp")):
            todo.append((rows, cols, bits, kw))
    if not todo:
        return
    import multiprocessing as mp
    n = workers or min(len(todo), max(1, (os.cpu_count() or 2) - 1))
    with mp.get_context("spawn").Pool(n) as pool:
        list(pool.imap_unordered(_build_one, todo))


def f32_activations(M, cols, seed=0, scale=1.0, outlier=True):
    """Full-mantissa f32 activations (NOT bf16-representable) with one outlier
    column 64x larger: exercises the hi/lo split and the per-token scaling."""
    rng = np.random.default_rng(7000 + seed)
    x = (rng.standard_normal((M, cols)) * scale).astype(np.float32)
    if outlier:
        x[:, (seed * 7919) % cols] *= 64.0
    return x
