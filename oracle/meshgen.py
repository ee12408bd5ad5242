"""CHECKER / BASELINE INFRASTRUCTURE -- never on the product path.

numpy restatement of the BASELINE.json mesh generator (`dgb_mesh_rectangle`,
paper_1502_02941_b200/csrc/host_mesh.cpp): the raw input (nodes, CCW elements, Dirichlet and
Neumann boundary pairs) that the reference's own `build_mesh` (mesh.cpp:51-187) turns into a
`Mesh`.  It lets `bench.py --impl reference` and the CPU-baseline timings feed the reference
(oracle/_ref) without loading the repo's CUDA library.  Bit-identical to the C++ generator
(tests/test_meshgen.py).

* nodes row-major over (i, j), x = lx * (i / nx); interior nodes jittered by
  (2 U - 1) * jitter * h per coordinate from splitmix64(jitter_seed), x then y per node;
* cell (i, j): lower (v00, v10, v11) and upper (v00, v11, v01) triangles, both CCW;
* permute: Fisher-Yates over the element list, k = splitmix64(permute_seed) % (i + 1);
* boundary pairs in the order y = 0, y = ly, x = 0, x = lx; side bits 4, 8, 1, 2 select Neumann.
"""
from __future__ import annotations

import numpy as np

MASK = (1 << 64) - 1


def _splitmix_stream(seed: int, n: int) -> np.ndarray:
    """The first n outputs of splitmix64(seed) as uint64."""
    with np.errstate(over="ignore"):
        k = np.arange(1, n + 1, dtype=np.uint64)
        z = np.uint64(seed & MASK) + k * np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def rectangle_raw(nx: int, ny: int, lx: float = 1.0, ly: float = 1.0, jitter: float = 0.0,
                  jitter_seed: int = 0, permute: bool = False, permute_seed: int = 0,
                  neumann_sides: int = 0) -> dict:
    px, py = nx + 1, ny + 1
    i = np.tile(np.arange(px, dtype=np.float64), py)
    j = np.repeat(np.arange(py, dtype=np.float64), px)
    x = lx * (i / nx)
    y = ly * (j / ny)
    if jitter > 0.0:
        interior = (i > 0) & (i < nx) & (j > 0) & (j < ny)
        n_int = int(interior.sum())
        u = (_splitmix_stream(jitter_seed, 2 * n_int) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
        hx, hy = lx / nx, ly / ny
        x[interior] = x[interior] + (2.0 * u[0::2] - 1.0) * (jitter * hx)
        y[interior] = y[interior] + (2.0 * u[1::2] - 1.0) * (jitter * hy)
    nodes = np.stack([x, y], axis=1)

    ci = np.tile(np.arange(nx, dtype=np.int64), ny)
    cj = np.repeat(np.arange(ny, dtype=np.int64), nx)
    v00 = cj * px + ci
    v10, v01, v11 = v00 + 1, v00 + px, v00 + px + 1
    elements = np.empty((2 * nx * ny, 3), np.int32)
    elements[0::2] = np.stack([v00, v10, v11], axis=1)
    elements[1::2] = np.stack([v00, v11, v01], axis=1)
    if permute:
        ne = elements.shape[0]
        draws = _splitmix_stream(permute_seed, ne - 1)
        ks = (draws % np.arange(ne, 1, -1, dtype=np.uint64)).astype(np.int64)  # i = ne-1 .. 1
        order = np.arange(ne, dtype=np.int64)
        for t, ii in enumerate(range(ne - 1, 0, -1)):
            k = ks[t]
            order[ii], order[k] = order[k], order[ii]
        elements = elements[order]

    def side(i0, j0, di, dj, count):
        s = np.arange(count, dtype=np.int64)
        a = (j0 + s * dj) * px + (i0 + s * di)
        b = (j0 + (s + 1) * dj) * px + (i0 + (s + 1) * di)
        return np.stack([a, b], axis=1).astype(np.int32)

    dirichlet, neumann = [], []
    for bit, args in ((4, (0, 0, 1, 0, nx)), (8, (0, ny, 1, 0, nx)), (1, (0, 0, 0, 1, ny)),
                      (2, (nx, 0, 0, 1, ny))):
        (neumann if neumann_sides & bit else dirichlet).append(side(*args))
    cat = lambda l: np.concatenate(l) if l else np.zeros((0, 2), np.int32)  # noqa: E731
    return {"nodes": nodes, "elements": elements, "dirichlet": cat(dirichlet),
            "neumann": cat(neumann)}


def unit_square_raw(n: int, jitter: float = 0.0, jitter_seed: int = 0, permute: bool = False,
                    permute_seed: int = 0, neumann_sides: int = 0) -> dict:
    return rectangle_raw(n, n, 1.0, 1.0, jitter, jitter_seed, permute, permute_seed,
                         neumann_sides)


def config_raw(cfg, n: int | None = None) -> dict:
    """Raw input of a BASELINE config's mesh (cfg: problems.Config), optionally at n x n."""
    from paper_1502_02941_b200.problems import SEED_JITTER, SEED_PERMUTE
    return unit_square_raw(cfg.n if n is None else n, cfg.jitter, SEED_JITTER, cfg.permute,
                           SEED_PERMUTE, cfg.neumann_sides)
