"""Seeded adversarial fuzz cases (plain numpy; shared by tests/test_gpu_fuzz.py,
tests/test_oracle_golden.py and tests/golden/make_golden.py ``fuzz``).

``case_arrays(seed)`` returns the raw inputs -- unnormalised quaternions
included, so the reference, the oracle and the GPU path all start from the
same bits.  Every case mixes Gaussians straddling the near plane and behind
the camera, exact position duplicates (depth ties), footprints from sub-pixel
to whole-image, opacities at 0, at 1 and within 1e-9 of the alpha floor,
splats on pixel centres, rotated off-centre cameras of 1-400 pixels per side,
E in {2, 3, 7, 40} with iid or block masks, and seven blend-floor settings."""

import numpy as np

BLENDS = [(1.0 / 255.0, 1e-4), (0.0, 0.0), (0.05, 1e-4), (1.0 / 255.0, 0.3), (0.0, 1e-4),
          (1.0 / 255.0, 0.0), (0.2, 0.5)]
N_CASES = 160


def _rotation(rng):
    q = rng.normal(size=4)
    w, x, y, z = q / np.linalg.norm(q)
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                     [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                     [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])


def _camera_row(rng):
    """[W, H, fx, fy, cx, cy, near, w2c(16)] (the golden camera-row layout)."""
    hi = 121 if rng.random() < 0.8 else 401
    W, H = int(rng.integers(1, hi)), int(rng.integers(1, hi))
    fx, fy = rng.uniform(20, 400), rng.uniform(20, 400)
    cx, cy = rng.uniform(-10, W + 10), rng.uniform(-10, H + 10)
    R = _rotation(rng) if rng.random() < 0.7 else np.eye(3)
    t = rng.normal(scale=0.3, size=3)
    w2c = np.eye(4)
    w2c[:3, :3], w2c[:3, 3] = R, t
    return np.concatenate([[W, H, fx, fy, cx, cy, 0.01], w2c.ravel()])


def case_arrays(seed):
    rng = np.random.default_rng(1000 + seed)
    cams = [_camera_row(rng) for _ in range(int(rng.integers(1, 4)))]
    W0, H0, fx0, fy0, cx0, cy0 = cams[0][:6]
    w2c0 = cams[0][7:].reshape(4, 4)
    n = int(rng.choice([1, 2, 17, 300, 1500, 3000, 20000]))
    # camera-space points inside / around the first view's frustum
    z = rng.uniform(0.3, 6.0, n)
    u = rng.uniform(-0.2 * W0, 1.2 * W0, n)
    v = rng.uniform(-0.2 * H0, 1.2 * H0, n)
    kind = rng.random(n)
    z = np.where(kind < 0.05, 0.01 + rng.normal(scale=1e-3, size=n), z)      # at the near plane
    z = np.where((kind >= 0.05) & (kind < 0.08), -rng.uniform(0.1, 2, n), z)  # behind
    on_px = (kind >= 0.08) & (kind < 0.15)                                    # on pixel centres
    u = np.where(on_px, np.floor(u) + 0.5, u)
    v = np.where(on_px, np.floor(v) + 0.5, v)
    pc = np.stack([(u - cx0) * z / fx0, (v - cy0) * z / fy0, z], axis=1)
    means = (pc - w2c0[:3, 3]) @ w2c0[:3, :3]  # camera -> world
    if n > 4:  # exact duplicates: equal depths in every view, tie order by id
        k = max(1, n // 10)
        src = rng.integers(0, n, k)
        dst = rng.integers(0, n, k)
        means[dst] = means[src]
    # footprints from sub-pixel to a few tens of pixels, anisotropic; 1% cover the image
    px = np.abs(z) / fx0
    scales = px[:, None] * np.exp(rng.uniform(np.log(0.05), np.log(12.0), (n, 3)))
    big = rng.random(n) < 0.01
    scales[big] *= rng.uniform(10, 100, (int(big.sum()), 1))
    quats = rng.normal(size=(n, 4)) * rng.uniform(0.1, 10, (n, 1))
    op = rng.uniform(0, 1, n)
    ok = rng.random(n)
    op = np.where(ok < 0.05, 1.0, op)
    op = np.where((ok >= 0.05) & (ok < 0.08), 0.0, op)
    near_floor = (ok >= 0.08) & (ok < 0.15)
    op = np.where(near_floor, (1.0 / 255.0) * (1 + rng.uniform(-1e-9, 1e-9, n)), op)
    E = int(rng.choice([2, 3, 7, 40]))
    masks = []
    for row in cams:
        w, h = int(row[0]), int(row[1])
        if rng.random() < 0.5:
            m = rng.integers(0, E, (h, w))
        else:
            bx = max(1, w // int(rng.integers(1, 5)))
            by = max(1, h // int(rng.integers(1, 5)))
            yy, xx = np.mgrid[0:h, 0:w]
            m = ((xx // bx) * 7 + (yy // by) * 3) % E
        masks.append(m.astype(np.uint16))
    af, tf = BLENDS[seed % len(BLENDS)]
    gamma = float(rng.choice([0.0, 0.1, 0.5, 0.95]))
    return dict(means=means, quats=quats, scales=scales, opac=op, cams=cams, masks=masks, E=E,
                floors=(af, tf), gamma=gamma)


def render_extras(seed, n, E):
    """Per-case render inputs: a 3-channel property, a one-object-per-Gaussian
    membership and tau."""
    rng = np.random.default_rng(7 + seed)
    ch = rng.random((n, 3))
    memb = np.zeros((E, n), np.uint8)
    memb[rng.integers(0, E, n), np.arange(n)] = 1
    tau = float(rng.choice([0.05, 0.3, 0.7]))
    return ch, memb, tau


def digest(c):
    """sha256 of a case's inputs (pins the generator across numpy versions)."""
    import hashlib
    h = hashlib.sha256()
    for k in ("means", "quats", "scales", "opac"):
        h.update(np.ascontiguousarray(c[k]).tobytes())
    for r, m in zip(c["cams"], c["masks"]):
        h.update(np.ascontiguousarray(r).tobytes())
        h.update(np.ascontiguousarray(m).tobytes())
    h.update(repr((c["E"], c["floors"], c["gamma"])).encode())
    return h.hexdigest()


def ambiguous_mask_pixels(oracle, means, quats, scales, opac, cam, memb, tau, floors, rel=1e-9):
    """Pixels where render_scene_mask's decision (maskrender.py:83-94) is within
    ``rel`` of flipping -- some object's alpha within rel of tau, or the two
    nearest qualified objects' blended depths within rel of each other (e.g.
    duplicated Gaussians in different objects) -- so float64 exp / BLAS
    rounding (~1e-16) can decide it.  ``oracle`` is the oracle module; ``cam``
    an oracle camera."""
    alphas, depths = [], []
    for obj in range(1, memb.shape[0]):
        _, a, d = oracle.render_view(means, quats, scales, opac, cam, None,
                                     memb[obj].astype(bool), floors[0], floors[1])
        alphas.append(a)
        depths.append(d)
    if not alphas:
        return np.zeros((cam.height, cam.width), bool)
    alphas, depths = np.array(alphas), np.array(depths)
    near_tau = (np.abs(alphas - tau) <= rel * tau).any(axis=0)
    q = np.where(alphas > tau * (1 - rel), depths, np.inf)
    q.sort(axis=0)
    if q.shape[0] < 2:
        return near_tau
    with np.errstate(invalid="ignore"):  # inf - inf where fewer than two qualify
        tie = np.isfinite(q[1]) & (np.abs(q[1] - q[0]) <= rel * np.abs(q[0]))
    return near_tau | tie


def label_band(oracle, values, gamma, scene_mode, rtol=1e-4, atol=1e-6):
    """Gaussians whose biased decision margin lies inside the north-star
    tolerance (flips there are exempt)."""
    total = np.asarray(values, np.float64).sum(axis=0)
    margin = oracle.decision_margin(values, gamma)
    band = np.abs(margin) <= 4 * (rtol + atol / np.maximum(total, 1e-30))
    return band.any(axis=0) if scene_mode else band[1]


PLY_VALUES = [np.nan, np.inf, -np.inf, 0.0, -0.0, 1e-45, 3e38, -3e38, 88.7, 710.0, -750.0,
              800.0, -800.0, 1e-30]


def ply_edits(seed, n_vertices, names):
    """Random value edits [(vertex, property, float32 value)] for a PLY record
    table: special values (NaN, +-inf, +-0, denormal, float32 extremes, exp
    overflow / underflow arguments, huge logits) dropped into random
    properties, and sometimes a zeroed or tiny quaternion."""
    rng = np.random.default_rng(5000 + seed)
    edits = []
    for _ in range(int(rng.integers(1, 6))):
        v = int(rng.integers(0, n_vertices))
        if rng.random() < 0.2:
            val = 0.0 if rng.random() < 0.5 else 1e-30
            edits += [(v, f"rot_{k}", val) for k in range(4)]
        else:  # half of the edits hit the activated properties
            hot = [q for q in names if q.startswith(("scale_", "rot_")) or q == "opacity"]
            prop = str(rng.choice(hot if rng.random() < 0.5 else names))
            edits.append((v, prop, float(rng.choice(PLY_VALUES))))
    return edits


def patch_ply(raw, edits):
    """Binary little-endian PLY bytes with record values overwritten."""
    raw = bytes(raw)
    head_end = raw.index(b"end_header\n") + len(b"end_header\n")
    names = [ln.split()[2] for ln in raw[:head_end].decode().splitlines()
             if ln.startswith("property")]
    rec = np.frombuffer(raw[head_end:], dtype=np.dtype([(p, "<f4") for p in names])).copy()
    with np.errstate(over="ignore"):
        for v, p, val in edits:
            rec[p][v] = np.float32(val)
    return raw[:head_end] + rec.tobytes(), names
