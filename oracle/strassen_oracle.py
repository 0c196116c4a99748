"""CPU oracle for the FP64 Strassen / Strassen-Winograd path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
import this module, and only as the checker or the timed CPU baseline; the product path
(paper_2309_00628_b200) never touches it.

A numpy restatement of the reference package ``matmulkit`` (/root/reference/pkg/src):
the divide-and-conquer interpreter (kernels.py:269-315), the memory-lean schedule
interpreter (schedules.py:249-297), the padding driver (hybrid.py:105-146) and the
closed-form cost models (kernels.py:204-249, schedules.py:215-246). It issues the same
numpy operations in the same order as the reference (np.matmul leaves, np.add /
np.subtract block sums into freshly allocated temporaries), so on identical inputs its
results are bit-identical to the reference's; tests/test_oracle_golden.py pins that against
golden vectors produced by the reference itself (tests/golden/make_golden.py).

The reference's straight-line micro kernels for orders <= 8 (microkernels.py) are
bit-identical to its literal recursion (asserted by the reference's own tests,
test_kernels.py:198-214); the oracle always runs the literal recursion.
"""
from __future__ import annotations

import numpy as np

# ---- step tables (reference kernels.py:66-160), tuple form ----------------------------
STRASSEN = (
    ("add", "SA1", "A11", "A22"), ("add", "SB1", "B11", "B22"), ("mul", "P1", "SA1", "SB1"),
    ("add", "SA2", "A21", "A22"), ("mul", "P2", "SA2", "B11"), ("sub", "SB3", "B12", "B22"),
    ("mul", "P3", "A11", "SB3"), ("sub", "SB4", "B21", "B11"), ("mul", "P4", "A22", "SB4"),
    ("add", "SA5", "A11", "A12"), ("mul", "P5", "SA5", "B22"), ("sub", "SA6", "A21", "A11"),
    ("add", "SB6", "B11", "B12"), ("mul", "P6", "SA6", "SB6"), ("sub", "SA7", "A12", "A22"),
    ("add", "SB7", "B21", "B22"), ("mul", "P7", "SA7", "SB7"), ("add", "C11", "P1", "P4"),
    ("sub", "C11", "C11", "P5"), ("add", "C11", "C11", "P7"), ("add", "C12", "P3", "P5"),
    ("add", "C21", "P2", "P4"), ("add", "C22", "P1", "P3"), ("sub", "C22", "C22", "P2"),
    ("add", "C22", "C22", "P6"),
)
WINOGRAD_BLOCK = (
    ("add", "S1", "A21", "A22"), ("sub", "S2", "S1", "A11"), ("sub", "S3", "A11", "A21"),
    ("sub", "T1", "B12", "B11"), ("sub", "T2", "B22", "T1"), ("sub", "T3", "B22", "B12"),
    ("sub", "S4", "A12", "S2"), ("sub", "T4", "T2", "B21"), ("mul", "P1", "A11", "B11"),
    ("mul", "P2", "A12", "B21"), ("mul", "P3", "S4", "B22"), ("mul", "P4", "A22", "T4"),
    ("mul", "P5", "S1", "T1"), ("mul", "P6", "S2", "T2"), ("mul", "P7", "S3", "T3"),
    ("add", "C11", "P1", "P2"), ("add", "U2", "P1", "P6"), ("add", "U3", "U2", "P7"),
    ("add", "U4", "U2", "P5"), ("add", "C12", "U4", "P3"), ("sub", "C21", "U3", "P4"),
    ("add", "C22", "U3", "P5"),
)
WINOGRAD_KNUTH = (
    ("add", "SCD", "A21", "A22"), ("sub", "SCDA", "SCD", "A11"), ("sub", "TCD", "B12", "B22"),
    ("sub", "TADC", "B11", "TCD"), ("sub", "SCA", "A21", "A11"), ("sub", "TCA", "B12", "B11"),
    ("add", "SAB", "A11", "A12"), ("sub", "SABCD", "SAB", "SCD"), ("sub", "TBCAD", "B21", "TADC"),
    ("mul", "M1", "A11", "B11"), ("mul", "M2", "A12", "B21"), ("mul", "MU", "SCA", "TCD"),
    ("mul", "MV", "SCD", "TCA"), ("mul", "MW", "SCDA", "TADC"), ("mul", "M6", "SABCD", "B22"),
    ("mul", "M7", "A22", "TBCAD"), ("add", "W", "M1", "MW"), ("add", "WU", "W", "MU"),
    ("add", "C11", "M1", "M2"), ("add", "C12", "W", "MV"), ("add", "C12", "C12", "M6"),
    ("add", "C21", "WU", "M7"), ("add", "C22", "WU", "MV"),
)
WINOGRAD_KNUTH_8CALL = WINOGRAD_KNUTH[:18] + (("mul", "M1B", "A11", "B11"), ("add", "C11", "M1B", "M2")) + \
    WINOGRAD_KNUTH[19:]
TABLES = {"strassen": STRASSEN, "winograd-block": WINOGRAD_BLOCK, "winograd-knuth": WINOGRAD_KNUTH,
          "winograd-knuth-8call": WINOGRAD_KNUTH_8CALL}

# ---- schedules (reference schedules.py:62-112): (symbol, op, lhs, rhs, store) ----------
TWO_TEMP = (
    ("S3", "-", "A11", "A21", "X"), ("T3", "-", "B22", "B12", "Y"), ("P7", "*", "S3", "T3", "C21"),
    ("S1", "+", "A21", "A22", "X"), ("T1", "-", "B12", "B11", "Y"), ("P5", "*", "S1", "T1", "C22"),
    ("S2", "-", "S1", "A11", "X"), ("T2", "-", "B22", "T1", "Y"), ("P6", "*", "S2", "T2", "C12"),
    ("S4", "-", "A12", "S2", "X"), ("P3", "*", "S4", "B22", "C11"), ("P1", "*", "A11", "B11", "X"),
    ("U2", "+", "P1", "P6", "C12"), ("U3", "+", "U2", "P7", "C21"), ("U4", "+", "U2", "P5", "C12"),
    ("U7", "+", "U3", "P5", "C22"), ("U5", "+", "U4", "P3", "C12"), ("T4", "-", "T2", "B21", "Y"),
    ("P4", "*", "A22", "T4", "C11"), ("U6", "-", "U3", "P4", "C21"), ("P2", "*", "A12", "B21", "C11"),
    ("U1", "+", "P1", "P2", "C11"),
)
IN_PLACE = (
    ("S3", "-", "A11", "A21", "C11"), ("S1", "+", "A21", "A22", "A21"), ("T1", "-", "B12", "B11", "C22"),
    ("T3", "-", "B22", "B12", "B12"), ("P7", "*", "S3", "T3", "C21"), ("S2", "-", "S1", "A11", "C12"),
    ("P1", "*", "A11", "B11", "C11"), ("T2", "-", "B22", "T1", "B11"), ("P5", "*", "S1", "T1", "A11"),
    ("T4", "-", "T2", "B21", "C22"), ("P4", "*", "A22", "T4", "A21"), ("S4", "-", "A12", "S2", "A22"),
    ("P6", "*", "S2", "T2", "C22"), ("U2", "+", "P1", "P6", "C22"), ("P2", "*", "A12", "B21", "C12"),
    ("U1", "+", "P1", "P2", "C11"), ("U4", "+", "U2", "P5", "C12"), ("U3", "+", "U2", "P7", "C22"),
    ("U6", "-", "U3", "P4", "C21"), ("U7", "+", "U3", "P5", "C22"), ("P3", "*", "S4", "B22", "A12"),
    ("U5", "+", "U4", "P3", "C12"),
)
SCHEDULES = {"two-temp": (TWO_TEMP, ("X", "Y")), "in-place": (IN_PLACE, ())}


# ---- policies (reference kernels.py:26-57), as (kind, param) tuples ----------------------
def policy(kind: str, param: int | None = None):
    if kind == "scalar":
        return ("scalar", 1)
    if kind == "unrolled":
        return ("unrolled", 8 if param is None else param)
    if kind == "naive-cutoff":
        return ("naive-cutoff", 12 if param is None else param)
    raise ValueError(kind)


def _is_leaf(n: int, pol) -> str | None:
    kind, p = pol
    if n == 1:
        return "scalar"
    if kind == "naive-cutoff" and n <= p:
        return "naive"
    return None


# ---- numerics -------------------------------------------------------------------------
def naive(a: np.ndarray, b: np.ndarray, out: np.ndarray) -> None:
    """Leaf / direct product (reference kernels.py:258-264): np.matmul into out."""
    if out.dtype == np.result_type(a, b):
        np.matmul(a, b, out=out)
    else:
        out[:, :] = a @ b


def _quads(x: np.ndarray, h: int, tag: str, env: dict) -> None:
    env[tag + "11"], env[tag + "12"] = x[:h, :h], x[:h, h:]
    env[tag + "21"], env[tag + "22"] = x[h:, :h], x[h:, h:]


def dc(steps, a: np.ndarray, b: np.ndarray, c: np.ndarray, pol) -> None:
    """Recursive step-table interpreter (reference kernels.py:269-315)."""
    n = a.shape[0]
    leaf = _is_leaf(n, pol)
    if leaf == "scalar":
        c[0, 0] = a[0, 0] * b[0, 0]
        return
    if leaf == "naive":
        naive(a, b, c)
        return
    h = n // 2
    env: dict = {}
    _quads(a, h, "A", env)
    _quads(b, h, "B", env)
    _quads(c, h, "C", env)
    dt = np.result_type(a, b)
    for op, dst, x, y in steps:
        d = env.get(dst)
        if d is None:
            d = env[dst] = np.empty((h, h), dtype=dt)
        if op == "add":
            np.add(env[x], env[y], out=d)
        elif op == "sub":
            np.subtract(env[x], env[y], out=d)
        else:
            dc(steps, env[x], env[y], d, pol)


def _bindings(rows, clobber: bool):
    """Operand locations per schedule row (the reference's validate_schedule bindings)."""
    quads = ("A11", "A12", "A21", "A22", "B11", "B12", "B21", "B22")
    holds = {q: q for q in quads}
    home = dict(holds)
    out = []
    for sym, op, lhs, rhs, store in rows:
        locs = (home[lhs], home[rhs])
        if op == "*" and clobber:
            for loc in set(locs):
                v = holds[loc]
                holds[loc] = None
                if home.get(v) == loc:
                    del home[v]
        prev = holds.get(store)
        if prev is not None and home.get(prev) == store:
            del home[prev]
        holds[store] = sym
        home[sym] = store
        out.append(locs)
    return out


def sched(name: str, a: np.ndarray, b: np.ndarray, c: np.ndarray, pol) -> None:
    """Memory-lean schedule interpreter (reference schedules.py:249-297)."""
    rows, temps = SCHEDULES[name]
    n = a.shape[0]
    leaf = _is_leaf(n, pol)
    if leaf == "scalar":
        c[0, 0] = a[0, 0] * b[0, 0]
        return
    if leaf == "naive":
        naive(a, b, c)
        return
    h = n // 2
    env: dict = {}
    _quads(a, h, "A", env)
    _quads(b, h, "B", env)
    _quads(c, h, "C", env)
    dt = np.result_type(a, b)
    for (sym, op, _, _, store), (lloc, rloc) in zip(rows, _bindings(rows, name == "in-place")):
        d = env.get(store)
        if d is None:
            d = env[store] = np.empty((h, h), dtype=dt)
        if op == "+":
            np.add(env[lloc], env[rloc], out=d)
        elif op == "-":
            np.subtract(env[lloc], env[rloc], out=d)
        else:
            sched(name, env[lloc], env[rloc], d, pol)


def product(kernel: str, a: np.ndarray, b: np.ndarray, pol, in_place_ok: bool = False) -> np.ndarray:
    """C = A B for square power-of-two operands via one named kernel."""
    c = np.empty(a.shape, dtype=np.result_type(a, b))
    if kernel in TABLES:
        dc(TABLES[kernel], a, b, c, pol)
    elif kernel in SCHEDULES:
        if kernel == "in-place" and not in_place_ok:
            a, b = a.copy(), b.copy()
        sched(kernel, a, b, c, pol)
    elif kernel == "naive":
        naive(a, b, c)
    else:
        raise ValueError(kernel)
    return c


def next_pow2(n: int) -> int:
    return 1 if n <= 1 else 1 << (n - 1).bit_length()


def multiply(a: np.ndarray, b: np.ndarray, kernel: str, pol) -> np.ndarray:
    """Shape-agnostic driver (reference hybrid.py:105-146): pad to square 2^j, unpad."""
    m, k = a.shape
    n = b.shape[1]
    dt = np.result_type(a, b)
    if kernel == "naive":
        c = np.empty((m, n), dtype=dt)
        naive(a, b, c)
        return c
    t = next_pow2(max(m, k, n))
    if m == k == n == t:
        return product(kernel, a, b, pol)
    pa = np.zeros((t, t), dtype=a.dtype)
    pa[:m, :k] = a
    pb = np.zeros((t, t), dtype=b.dtype)
    pb[:k, :n] = b
    return product(kernel, pa, pb, pol, in_place_ok=True)[:m, :n].copy()


# ---- cost models (reference kernels.py:204-249, schedules.py:215-246) ------------------
def _peak(entries, hh, child, is_temp):
    live = peak = 0
    seen = set()
    for is_mul, dst in entries:
        if is_temp(dst) and dst not in seen:
            seen.add(dst)
            live += hh
            peak = max(peak, live)
        if is_mul:
            peak = max(peak, live + child)
    return peak


def cost(kernel: str, pol, n: int):
    """(mults, adds, buffer events, peak live aux elements) of the literal recursion."""
    kind, p = pol
    if n == 1:
        return (1, 0, 0, 0)
    if kind == "naive-cutoff" and n <= p:
        return (n ** 3, n * n * (n - 1), 0, 0)
    if kind == "unrolled" and n <= p:
        m, a, _, _ = cost("winograd-block" if kernel in SCHEDULES else kernel, ("scalar", 1), n)
        return (m, a, 0, 0)
    h = n // 2
    cm, ca, cb, cp = cost(kernel, pol, h)
    if kernel in SCHEDULES:
        rows, temps = SCHEDULES[kernel]
        entries = [(op == "*", store) for _, op, _, _, store in rows]
        peak = _peak(entries, h * h, cp, lambda d: d in temps)
        adds = sum(op != "*" for _, op, _, _, _ in rows)
        return (7 * cm, 7 * ca + adds * h * h, 7 * cb + len(temps), peak)
    steps = TABLES[kernel]
    cq = {"C11", "C12", "C21", "C22"}
    entries = [(op == "mul", dst) for op, dst, _, _ in steps]
    peak = _peak(entries, h * h, cp, lambda d: d not in cq)
    muls = sum(op == "mul" for op, *_ in steps)
    adds = sum(op != "mul" for op, *_ in steps)
    temps = len({d for _, d, _, _ in steps if d not in cq})
    return (muls * cm, muls * ca + adds * h * h, muls * cb + temps, peak)


# ---- seeded operands of BASELINE.json's configs ----------------------------------------
SEED = 20240901


def operands(cfg: int, seed: int = SEED, scale: int = 1):
    """A then B from one np.random.default_rng(seed) (reference metrics.py:62-68, 105-109).

    cfg 1, 3: uniform[-1, 1) squares (n = 256, 8192); cfg 2: integers in [-8, 8] as FP64
    (n = 1024); cfg 4: standard normal (n = 16384); cfg 5: uniform, 12000x14000 . 14000x10000.
    ``scale`` divides every extent (bounded CPU samples).
    """
    rng = np.random.default_rng(seed)
    if cfg == 1:
        n = 256 // scale
        return rng.uniform(-1.0, 1.0, (n, n)), rng.uniform(-1.0, 1.0, (n, n))
    if cfg == 2:
        n = 1024 // scale
        return (rng.integers(-8, 9, (n, n), dtype=np.int64).astype(np.float64),
                rng.integers(-8, 9, (n, n), dtype=np.int64).astype(np.float64))
    if cfg == 3:
        n = 8192 // scale
        return rng.uniform(-1.0, 1.0, (n, n)), rng.uniform(-1.0, 1.0, (n, n))
    if cfg == 4:
        n = 16384 // scale
        return rng.standard_normal((n, n)), rng.standard_normal((n, n))
    if cfg == 5:
        m, k, n = 12000 // scale, 14000 // scale, 10000 // scale
        return rng.uniform(-1.0, 1.0, (m, k)), rng.uniform(-1.0, 1.0, (k, n))
    raise ValueError(cfg)


def tolerance(n: int, amax: float, bmax: float, c: float = 1.0) -> float:
    """The stated normwise bound (BASELINE.json north_star):

        |C - C_ref|_max <= c * n^(log2 12) * u * |A|_max * |B|_max,  u = 2^-53, c = 1.

    (Higham's worst case for the Winograd form has exponent log2 18; log2 12 is the stated
    contract and holds with a wide margin in practice.)
    """
    return c * float(n) ** np.log2(12.0) * 2.0 ** -53 * amax * bmax


# ---- leaf-product decomposition (for the multi-GPU sharding checks) --------------------
def one_level_coefficients(kernel: str):
    """(a, b, c) one-level coefficient form of a step table, by symbolic execution."""
    steps = TABLES[kernel]
    env = {}
    for i, q in enumerate(("11", "12", "21", "22")):
        env["A" + q] = [int(j == i) for j in range(4)]
        env["B" + q] = [int(j == i) for j in range(4)]
    a, b = [], []
    nprod = sum(op == "mul" for op, *_ in steps)
    for op, dst, x, y in steps:
        if op == "mul":
            a.append(env[x])
            b.append(env[y])
            env[dst] = [int(j == len(a) - 1) for j in range(nprod)]
        else:
            s = 1 if op == "add" else -1
            env[dst] = [u + s * v for u, v in zip(env[x], env[y])]
    c = [env["C" + q] for q in ("11", "12", "21", "22")]
    return a, b, c


def leaf_partial(kernel: str, a: np.ndarray, b: np.ndarray, levels: int, first: int, count: int,
                 panels: int = 1) -> np.ndarray:
    """Sum of the contributions of shard units [first, first+count) to C; unit u is row panel
    (u mod panels) of leaf (u div panels), leaves in level-major order."""
    ca, cb, cc = one_level_coefficients(kernel)
    nprod = len(ca)
    n = a.shape[0]
    out = np.zeros((n, n), dtype=np.result_type(a, b))

    def rec(level, xs, ys, ds, size, index):
        # xs / ys / ds: lists of (row, col, sign) blocks of A / B / C at this size
        sub = nprod ** (levels - level) * panels
        if index * panels + sub <= first or index * panels >= first + count:
            return
        if level == levels:
            u0 = index * panels
            lo, hi = max(u0, first) - u0, min(u0 + panels, first + count) - u0
            pr = size // panels
            r0, r1 = lo * pr, hi * pr
            x = sum(s * a[r + r0:r + r1, c:c + size] for r, c, s in xs)
            y = sum(s * b[r:r + size, c:c + size] for r, c, s in ys)
            p = x @ y
            for r, c, s in ds:
                out[r + r0:r + r1, c:c + size] += s * p
            return
        h = size // 2
        off = [(0, 0), (0, h), (h, 0), (h, h)]
        for p in range(nprod):
            nx = [(r + off[q][0], c + off[q][1], s * ca[p][q]) for r, c, s in xs for q in range(4) if ca[p][q]]
            ny = [(r + off[q][0], c + off[q][1], s * cb[p][q]) for r, c, s in ys for q in range(4) if cb[p][q]]
            nd = [(r + off[q][0], c + off[q][1], s * cc[q][p]) for r, c, s in ds for q in range(4) if cc[q][p]]
            rec(level + 1, nx, ny, nd, h, index + p * nprod ** (levels - level - 1))

    rec(0, [(0, 0, 1)], [(0, 0, 1)], [(0, 0, 1)], n, 0)
    return out
