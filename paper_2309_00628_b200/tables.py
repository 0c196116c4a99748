"""Per-level algebra of the divide-and-conquer products, restated as data.

Each table is the reference's step table written in ordinary notation and parsed into
the reference's tuple form ``(op, dst, lhs, rhs)`` with op in {"add", "sub", "mul"}:

* STRASSEN_STEPS            reference kernels.py:66-92   (18 block adds, 7 products)
* WINOGRAD_BLOCK_STEPS      reference kernels.py:96-119  (15 block adds, 7 products)
* WINOGRAD_KNUTH_STEPS      reference kernels.py:128-152 (16 block adds, 7 products)
* WINOGRAD_KNUTH_8CALL_STEPS reference kernels.py:156-160 (M1 recomputed for C11)

The memory-lean schedules (paper Tables 2 and 3) are ``symbol = lhs op rhs -> store``:

* TWO_TEMP_ROWS  reference schedules.py:62-85
* IN_PLACE_ROWS  reference schedules.py:89-112

The same algebra is compiled natively by the engine (csrc/mk_engine.cu), which derives
one-level coefficient tables from these steps symbolically; ``coefficients`` below does
the same derivation in Python so the two can be cross-checked in tests.
"""
from __future__ import annotations

_OPS = {"+": "add", "-": "sub", "*": "mul"}


def _parse(text: str):
    steps = []
    for line in text.strip().splitlines():
        line = line.split("#")[0].strip()
        if not line:
            continue
        dst, expr = (p.strip() for p in line.split("="))
        lhs, sym, rhs = expr.split()
        steps.append((_OPS[sym], dst, lhs, rhs))
    return tuple(steps)


def _parse_schedule(text: str):
    rows = []
    for line in text.strip().splitlines():
        line = line.strip()
        if not line:
            continue
        body, store = (p.strip() for p in line.split("->"))
        sym, expr = (p.strip() for p in body.split("="))
        lhs, op, rhs = expr.split()
        rows.append((sym, op, lhs, rhs, store))
    return tuple(rows)


STRASSEN_STEPS = _parse("""
    SA1 = A11 + A22
    SB1 = B11 + B22
    P1  = SA1 * SB1
    SA2 = A21 + A22
    P2  = SA2 * B11
    SB3 = B12 - B22
    P3  = A11 * SB3
    SB4 = B21 - B11
    P4  = A22 * SB4
    SA5 = A11 + A12
    P5  = SA5 * B22
    SA6 = A21 - A11
    SB6 = B11 + B12
    P6  = SA6 * SB6
    SA7 = A12 - A22
    SB7 = B21 + B22
    P7  = SA7 * SB7
    C11 = P1 + P4
    C11 = C11 - P5
    C11 = C11 + P7
    C12 = P3 + P5
    C21 = P2 + P4
    C22 = P1 + P3
    C22 = C22 - P2
    C22 = C22 + P6
""")

WINOGRAD_BLOCK_STEPS = _parse("""
    S1 = A21 + A22
    S2 = S1 - A11
    S3 = A11 - A21
    T1 = B12 - B11
    T2 = B22 - T1
    T3 = B22 - B12
    S4 = A12 - S2
    T4 = T2 - B21
    P1 = A11 * B11
    P2 = A12 * B21
    P3 = S4 * B22
    P4 = A22 * T4
    P5 = S1 * T1
    P6 = S2 * T2
    P7 = S3 * T3
    C11 = P1 + P2
    U2 = P1 + P6
    U3 = U2 + P7
    U4 = U2 + P5
    C12 = U4 + P3
    C21 = U3 - P4
    C22 = U3 + P5
""")

WINOGRAD_KNUTH_STEPS = _parse("""
    SCD   = A21 + A22
    SCDA  = SCD - A11
    TCD   = B12 - B22
    TADC  = B11 - TCD
    SCA   = A21 - A11
    TCA   = B12 - B11
    SAB   = A11 + A12
    SABCD = SAB - SCD
    TBCAD = B21 - TADC
    M1 = A11 * B11
    M2 = A12 * B21
    MU = SCA * TCD
    MV = SCD * TCA
    MW = SCDA * TADC
    M6 = SABCD * B22
    M7 = A22 * TBCAD
    W  = M1 + MW
    WU = W + MU
    C11 = M1 + M2
    C12 = W + MV
    C12 = C12 + M6
    C21 = WU + M7
    C22 = WU + MV
""")

# the 8-call form evaluates A11*B11 a second time (M1B) for C11
WINOGRAD_KNUTH_8CALL_STEPS = (
    WINOGRAD_KNUTH_STEPS[:18] + (("mul", "M1B", "A11", "B11"), ("add", "C11", "M1B", "M2"))
    + WINOGRAD_KNUTH_STEPS[19:]
)

TWO_TEMP_ROWS = _parse_schedule("""
    S3 = A11 - A21 -> X
    T3 = B22 - B12 -> Y
    P7 = S3 * T3 -> C21
    S1 = A21 + A22 -> X
    T1 = B12 - B11 -> Y
    P5 = S1 * T1 -> C22
    S2 = S1 - A11 -> X
    T2 = B22 - T1 -> Y
    P6 = S2 * T2 -> C12
    S4 = A12 - S2 -> X
    P3 = S4 * B22 -> C11
    P1 = A11 * B11 -> X
    U2 = P1 + P6 -> C12
    U3 = U2 + P7 -> C21
    U4 = U2 + P5 -> C12
    U7 = U3 + P5 -> C22
    U5 = U4 + P3 -> C12
    T4 = T2 - B21 -> Y
    P4 = A22 * T4 -> C11
    U6 = U3 - P4 -> C21
    P2 = A12 * B21 -> C11
    U1 = P1 + P2 -> C11
""")

IN_PLACE_ROWS = _parse_schedule("""
    S3 = A11 - A21 -> C11
    S1 = A21 + A22 -> A21
    T1 = B12 - B11 -> C22
    T3 = B22 - B12 -> B12
    P7 = S3 * T3 -> C21
    S2 = S1 - A11 -> C12
    P1 = A11 * B11 -> C11
    T2 = B22 - T1 -> B11
    P5 = S1 * T1 -> A11
    T4 = T2 - B21 -> C22
    P4 = A22 * T4 -> A21
    S4 = A12 - S2 -> A22
    P6 = S2 * T2 -> C22
    U2 = P1 + P6 -> C22
    P2 = A12 * B21 -> C12
    U1 = P1 + P2 -> C11
    U4 = U2 + P5 -> C12
    U3 = U2 + P7 -> C22
    U6 = U3 - P4 -> C21
    U7 = U3 + P5 -> C22
    P3 = S4 * B22 -> A12
    U5 = U4 + P3 -> C12
""")

C_QUADS = frozenset({"C11", "C12", "C21", "C22"})
INPUT_QUADS = frozenset({"A11", "A12", "A21", "A22", "B11", "B12", "B21", "B22"})


def coefficients(steps):
    """One-level coefficient form of a step table (the engine derives the same natively).

    Returns (a, b, c): a[p] / b[p] are the +-1 coefficients of A / B quadrants (11, 12, 21,
    22) in product p's operands, c[q][p] the coefficient of product p in C quadrant q.
    """
    names = ("11", "12", "21", "22")
    env = {}
    for i, q in enumerate(names):
        env["A" + q] = ("A", tuple(int(j == i) for j in range(4)))
        env["B" + q] = ("B", tuple(int(j == i) for j in range(4)))
    a, b = [], []
    nprod = sum(1 for op, *_ in steps if op == "mul")
    for op, dst, x, y in steps:
        (kx, vx), (ky, vy) = env[x], env[y]
        if op == "mul":
            p = len(a)
            a.append(vx)
            b.append(vy)
            env[dst] = ("P", tuple(int(j == p) for j in range(nprod)))
        else:
            s = 1 if op == "add" else -1
            env[dst] = (kx, tuple(u + s * v for u, v in zip(vx, vy)))
    c = [list(env["C" + q][1]) for q in names]
    return a, b, c
