"""The C-ABI library: it loads, exports every function include/mk_strassen.h declares, and
its host-only planning entry points (no CUDA calls) behave as specified. CPU only."""
import ctypes
import os
import re

import pytest

from paper_2309_00628_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "mk_strassen.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(mk_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(_lib.LIB_PATH):
        import __graft_entry__

        __graft_entry__.build()
    return _lib.load()


def test_library_exports_every_declared_symbol(lib):
    names = declared_functions()
    assert len(names) >= 15
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(_lib.exported_symbols())


def test_version_and_options(lib):
    assert lib.mk_version() >= 2
    assert lib.mk_set_option(_lib.MK_OPT_FUSE_PREADDS, 0) == 0
    assert lib.mk_set_option(999, 1) == _lib.MK_ERR_ARG
    assert b"unknown option" in lib.mk_last_error()


def levels(lib, n, kind, param, algo):
    out = ctypes.c_int(-1)
    rc = lib.mk_levels_for_policy(n, kind, param, _lib.ALGO_IDS[algo], ctypes.byref(out))
    assert rc == 0
    return out.value


def test_levels_follow_reference_recursion(lib):
    # naive-cutoff: leaf when n <= threshold (kernels.py:276)
    assert levels(lib, 8192, 2, 1024, "winograd-block") == 3
    assert levels(lib, 16384, 2, 8192, "winograd-block") == 1
    assert levels(lib, 16384, 2, 4096, "winograd-block") == 2
    assert levels(lib, 1024, 2, 64, "strassen") == 4
    assert levels(lib, 256, 2, 32, "winograd-block") == 3
    assert levels(lib, 64, 2, 64, "winograd-block") == 0
    # scalar / unrolled recursion is clamped at the engine's minimum leaf order (32)
    assert levels(lib, 256, 0, 1, "strassen") == 3
    assert levels(lib, 16, 0, 1, "strassen") == 0
    assert levels(lib, 64, 1, 8, "winograd-block") == 1
    # at most 5 levels whatever the policy asks for
    assert levels(lib, 16384, 0, 1, "strassen") == 5
    assert levels(lib, 16384, 2, 32, "winograd-block") == 5
    # the storage maps of the memory-lean schedules stay observable on small orders
    assert levels(lib, 16, 0, 1, "in-place") == 1
    assert levels(lib, 2, 0, 1, "in-place") == 0


def test_workspace_sizes(lib):
    ws = lambda algo, n, L: lib.mk_workspace_bytes(_lib.ALGO_IDS[algo], n, L)  # noqa: E731
    # one level: no workspace at all (operands are materialised only when a sum is needed:
    # two slots of (n/2)^2 at the top level)
    assert ws("in-place", 1024, 1) == 0 and ws("in-place", 1024, 3) == 0
    assert ws("winograd-block", 1024, 1) == 2 * 512 * 512 * 8
    assert ws("two-temp", 1024, 1) == 2 * 512 * 512 * 8
    # deeper: two-temp keeps the paper's two (n/2^(l+1))^2 slots per literal level (default)
    assert ws("two-temp", 1024, 3) == 2 * 8 * (512 ** 2 + 256 ** 2 + 128 ** 2)
    assert ws("two-temp", 1024, 2) == 2 * 8 * (512 ** 2 + 256 ** 2) < ws("winograd-block", 1024, 2)
    assert ws("winograd-block", 16384, 1) == 2 * 8192 * 8192 * 8
    assert ws("winograd-block", 16, 5) == 0  # invalid (leaf order < 2)
    assert lib.mk_rect_workspace_bytes(_lib.ALGO_IDS["winograd-block"], 12000, 10000, 14000, 5) > 0


def test_plan_options_change_workspace_not_counts(lib):
    ws = lambda algo, n, L: lib.mk_workspace_bytes(_lib.ALGO_IDS[algo], n, L)  # noqa: E731
    try:
        assert lib.mk_set_option(_lib.MK_OPT_PLAN, 1) == 0  # depth-first: operand sums only
        assert ws("winograd-block", 16384, 2) == (2 * 8192 ** 2 + 2 * 4096 ** 2) * 8
        assert lib.mk_set_option(_lib.MK_OPT_PLAN, 2) == 0  # hybrid: one top-level subtree at a time
        hybrid = ws("winograd-block", 16384, 3)
        assert lib.mk_set_option(_lib.MK_OPT_PLAN, 0) == 0
        # breadth-first, default passes of 4 top-level products: at most the reference's own
        # modeled block-Winograd peak (4.97 n^2 elements, 9.9 GiB at n = 16384)
        assert ws("winograd-block", 16384, 2) <= 4.97 * 16384 ** 2 * 8
        assert lib.mk_set_option(_lib.MK_OPT_BFS_GROUP, 7) == 0  # one pass: every depth at once
        assert ws("winograd-block", 16384, 2) > 6 * 16384 ** 2 * 8
        assert hybrid * 4 < ws("winograd-block", 16384, 3)
        assert lib.mk_set_option(_lib.MK_OPT_BFS_GROUP, 9) == _lib.MK_ERR_ARG
        assert ws("two-temp", 16384, 2) == (2 * 8192 ** 2 + 2 * 4096 ** 2) * 8  # literal to the leaves
        assert lib.mk_set_option(_lib.MK_OPT_LITERAL_TAIL, 1) == 0  # breadth-first tail: more scratch
        assert ws("two-temp", 16384, 2) > (2 * 8192 ** 2 + 2 * 4096 ** 2) * 8
        assert lib.mk_set_option(_lib.MK_OPT_PLAN, 7) == _lib.MK_ERR_ARG
    finally:
        lib.mk_set_option(_lib.MK_OPT_PLAN, 0)
        lib.mk_set_option(_lib.MK_OPT_LITERAL_TAIL, 0)
        lib.mk_set_option(_lib.MK_OPT_BFS_GROUP, 0)


def test_product_counts(lib):
    assert lib.mk_product_count(_lib.ALGO_IDS["winograd-block"], 2) == 49
    assert lib.mk_product_count(_lib.ALGO_IDS["winograd-knuth-8call"], 1) == 8
    assert lib.mk_product_count(_lib.ALGO_IDS["two-temp"], 1) == -1


def test_plain_c_consumer_links_and_runs(lib, tmp_path):
    """include/mk_strassen.h is a usable C boundary: a C program links the .so (no Python)."""
    import shutil
    import subprocess

    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    exe = tmp_path / "abi_check"
    src = os.path.join(ROOT, "tests", "c", "abi_check.c")
    libdir = os.path.dirname(_lib.LIB_PATH)
    subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), src, "-o", str(exe),
                    "-L", libdir, "-lmk_strassen", f"-Wl,-rpath,{libdir}"], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=60)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "abi_check ok" in out.stdout


def test_thread_plan_override_is_per_thread(lib):
    """mk_set_thread_option: the sizing and the launch of one call see the calling thread's plan,
    whatever another thread sets process-wide in between (device.py _memory_aware_plan)."""
    import threading

    ws = lambda n, L: lib.mk_workspace_bytes(_lib.ALGO_IDS["winograd-block"], n, L)  # noqa: E731
    dfs = (2 * 8192 ** 2 + 2 * 4096 ** 2) * 8
    seen = {}
    try:
        assert lib.mk_set_thread_option(_lib.MK_OPT_PLAN, 1) == 0
        assert ws(16384, 2) == dfs

        def other():
            seen["other_before"] = ws(16384, 2)  # no override in this thread: breadth-first
            lib.mk_set_option(_lib.MK_OPT_PLAN, 2)  # process-wide change by another thread
            seen["other_after"] = ws(16384, 3)

        t = threading.Thread(target=other)
        t.start()
        t.join()
        assert seen["other_before"] > dfs
        assert ws(16384, 2) == dfs  # this thread's override still wins
        v = ctypes.c_int(-1)
        assert lib.mk_get_option(_lib.MK_OPT_PLAN, ctypes.byref(v)) == 0 and v.value == 1
        assert lib.mk_set_thread_option(_lib.MK_OPT_PLAN, -1) == 0
        assert lib.mk_get_option(_lib.MK_OPT_PLAN, ctypes.byref(v)) == 0 and v.value == 2
        assert lib.mk_set_thread_option(_lib.MK_OPT_PLAN, 5) == _lib.MK_ERR_ARG
        assert lib.mk_set_thread_option(_lib.MK_OPT_LEAF_SLICES, 8) == _lib.MK_ERR_ARG
    finally:
        lib.mk_set_thread_option(_lib.MK_OPT_PLAN, -1)
        lib.mk_set_thread_option(_lib.MK_OPT_LITERAL_TAIL, -1)
        lib.mk_set_option(_lib.MK_OPT_PLAN, 0)


def test_option_enum_matches_the_binding_and_round_trips_without_a_gpu():
    """include/mk_strassen.h's `enum mk_option` and _lib.py's MK_OPT_* constants name the same keys
    with the same values; the launch-shape options (MK_OPT_PDL, MK_OPT_PIPELINE) are plain process
    settings, so they round-trip through mk_set_option / mk_get_option with no device present."""
    import re

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    text = open(os.path.join(root, "include", "mk_strassen.h")).read()
    body = re.search(r"enum mk_option \{(.*?)\};", text, re.S).group(1)
    header = {k: int(v) for k, v in re.findall(r"(MK_OPT_\w+)\s*=\s*(\d+)", body)}
    binding = {k: v for k, v in vars(_lib).items() if k.startswith("MK_OPT_")}
    assert header == binding and len(set(header.values())) == len(header)
    lib = _lib.load(required=True)
    v = ctypes.c_int(-1)
    for key, default, other in ((_lib.MK_OPT_PDL, 1, 0), (_lib.MK_OPT_PIPELINE, 1, 2), (_lib.MK_OPT_PIPELINE, 1, 0)):
        assert lib.mk_get_option(key, ctypes.byref(v)) == 0 and v.value == default
        try:
            assert lib.mk_set_option(key, other) == 0
            assert lib.mk_get_option(key, ctypes.byref(v)) == 0 and v.value == other
        finally:
            assert lib.mk_set_option(key, default) == 0
    assert lib.mk_set_option(_lib.MK_OPT_PIPELINE, 3) == _lib.MK_ERR_ARG
    assert lib.mk_set_option(_lib.MK_OPT_PIPELINE, -1) == _lib.MK_ERR_ARG
