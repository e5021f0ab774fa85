"""CPU-side checks of the boundary (`-m "not gpu"`): the C-ABI library loads
and exports every symbol include/*.h declares, argument errors are caught on
the host, and the product and the oracle share no code."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2410_17226_b200", "libcbfs.so")


def declared(header):
    txt = open(os.path.join(ROOT, "include", header)).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(cbfs_\w+|cg_\w+)\s*\(", txt, flags=re.M)))


def test_library_built_and_exports_all_symbols():
    if not os.path.exists(LIB):
        import __graft_entry__
        __graft_entry__.build()
    lib = ctypes.CDLL(LIB)
    names = declared("cbfs.h")
    assert len(names) >= 14, names
    for name in names:
        assert hasattr(lib, name), f"libcbfs.so does not export {name}"


def test_generator_library_exports_all_symbols():
    import cbfs_inputs
    lib = ctypes.CDLL(cbfs_inputs.build())
    for name in declared("cbfs_gen.h"):
        assert hasattr(lib, name), name


def test_host_side_argument_errors():
    import paper_2410_17226_b200 as cb
    lib = cb._lib
    assert lib.cbfs_graph_create(4, None, None, 0, 0, 0, None, None) == cb.CBFS_EINVAL
    assert lib.cbfs_run(None, None, None, 0, 2, 2, None, None, 3, None, 0, None) == cb.CBFS_EINVAL
    assert lib.cbfs_select_clusters(None, 1, 64, 2, 0, 0, None, None, None, None) == cb.CBFS_EINVAL
    assert lib.cbfs_decode(10, 1, 2, 3, None, 2, None, 0, 1, None, None) == cb.CBFS_EINVAL
    assert lib.cbfs_query_distance(10, 1, 2, 5, ctypes.c_void_p(8), 2, ctypes.c_void_p(8), ctypes.c_void_p(8),
                                   None, None, 0, None, None) == cb.CBFS_EINVAL  # planes must be d or d+1
    assert lib.cbfs_set_direction_alpha(ctypes.c_double(0.0)) == cb.CBFS_EINVAL
    assert b"alpha" in lib.cbfs_last_error()
    h = ctypes.c_void_p()
    fake = ctypes.c_void_p(8)
    # the NEXT-row entry points: host-side argument checks before any device work
    assert lib.cbfs_labels_build_w(None, None, None, 0, 2, 2, 64, ctypes.byref(h), None) == cb.CBFS_EINVAL
    assert lib.cbfs_run_wide(None, None, None, 1, 3, 2, 2, None, None, 3, None, 0, None) == cb.CBFS_EUNSUPPORTED
    assert b"words" in lib.cbfs_last_error()
    assert lib.cbfs_run_wide(None, None, None, 1, 2, 2, 2, None, None, 3, None, 0, None) == cb.CBFS_EINVAL
    assert lib.cbfs_select_clusters_wide(None, 1, 100, 2, 0, 0, 3, fake, fake, ctypes.byref(ctypes.c_uint32()),
                                         None) == cb.CBFS_EUNSUPPORTED
    assert lib.cbfs_select_clusters_wide(None, 1, 200, 2, 0, 0, 2, fake, fake, ctypes.byref(ctypes.c_uint32()),
                                         None) == cb.CBFS_EINVAL  # k > 64 * words
    assert lib.cbfs_decode_wide(10, 1, 2, 2, 3, fake, 2, fake, 0, 129, fake, None) == cb.CBFS_EINVAL  # k > 128
    assert lib.cbfs_query_distance_wide(10, 1, 3, 2, 3, fake, 2, fake, fake, fake, fake, 1, fake,
                                        None) == cb.CBFS_EUNSUPPORTED
    assert lib.cbfs_pll_build(None, None, None, 0, 2, 200, 1000, 256, ctypes.byref(h), None) == cb.CBFS_EINVAL
    assert lib.cbfs_pll_query(None, fake, fake, 1, fake, None) == cb.CBFS_EINVAL
    assert lib.cbfs_pll_destroy(None) == cb.CBFS_OK
    # output consumers / per-round statistics (host-side checks)
    assert lib.cbfs_run_digest(None, None, None, 0, 2, 2, 3, None, None, 0, None) == cb.CBFS_EINVAL
    assert lib.cbfs_run_rounds(None, None, None, 0, 2, None, 8, None, 0, None) == cb.CBFS_EINVAL
    assert lib.cbfs_digest_store(10, 1, 3, fake, 3, fake, fake, None) == cb.CBFS_EINVAL  # dist_bytes
    assert lib.cbfs_digest_store(10, 1, 3, fake, 2, None, fake, None) == cb.CBFS_EINVAL  # null masks
    assert lib.cbfs_digest_store(10, 0, 3, None, 2, None, None, None) == cb.CBFS_OK  # nothing to do
    # n must stay below 2^26 (packed (vertex, lane) entries never equal the all-ones sentinel)
    assert lib.cbfs_graph_create(1 << 26, fake, fake, 1, 0, 0, None, ctypes.byref(h)) == cb.CBFS_EUNSUPPORTED
    assert cb.CBFS_MAX_N == (1 << 26) - 1
    assert cb.cbfs_version().startswith("cbfs-b200")


def test_budget_arithmetic_in_the_library():
    """K12 budget arithmetic through the C-ABI against the
    paper-printed values of tests/golden/budget.txt (record bytes and cluster
    counts at t = 1,024 B/vertex)."""
    import paper_2410_17226_b200 as cb
    rows = [ln.split() for ln in open(os.path.join(ROOT, "tests", "golden", "budget.txt"))
            if ln.strip() and not ln.startswith("#")]
    assert rows
    for t, w, d, rb, r, *_ in rows:
        assert cb.cbfs_record_bytes(int(w), int(d), 1) == int(rb)
        assert cb.cbfs_budget_clusters(int(t), int(w), int(d), 1) == int(r)
    assert cb.cbfs_record_bytes(0, 2, 1) == 1  # plain landmark: Delta alone
    assert cb.cbfs_record_bytes(64, 2, 2) == 18
    with pytest.raises(cb.CbfsError):
        cb.cbfs_record_bytes(12, 2, 1)


def _sources(dirpath, exts):
    for dp, _, fs in os.walk(dirpath):
        for f in fs:
            if f.endswith(exts):
                yield os.path.join(dp, f)


def _deps(path):
    """#include targets, imports and dlopen'd library names of a source file."""
    txt = open(path).read()
    inc = re.findall(r'^\s*#\s*include\s*[<"]([^>"]+)[>"]', txt, flags=re.M)
    imp = re.findall(r"^\s*(?:from\s+([\w\.]+)\s+import|import\s+([\w\.]+))", txt, flags=re.M)
    libs = re.findall(r"(lib\w+\.so)", txt)
    return inc + [a or b for a, b in imp] + libs


def test_product_and_oracle_share_no_code():
    prod = list(_sources(os.path.join(ROOT, "paper_2410_17226_b200"), (".py", ".cu", ".cuh", ".h", ".c")))
    orc = list(_sources(os.path.join(ROOT, "oracle"), (".py", ".c", ".h")))
    assert prod and orc
    for p in prod:
        for dep in _deps(p):
            assert "oracle" not in dep and "cbfs_inputs" not in dep and "cbfs_gen" not in dep, (p, dep)
    for p in orc:
        for dep in _deps(p):
            assert "paper_2410_17226_b200" not in dep and "libcbfs.so" != dep and "cbfs.h" not in dep, (p, dep)


def test_bench_and_smoke_only_oracle_users():
    """Only tests/, __graft_entry__.py and bench.py may touch oracle/."""
    for p in _sources(ROOT, (".py",)):
        rel = os.path.relpath(p, ROOT)
        if rel.startswith(("tests", "oracle", "baseline", "build")) or rel in ("__graft_entry__.py", "bench.py"):
            continue
        txt = open(p).read()
        assert not re.search(r"^\s*(import oracle|from oracle)", txt, flags=re.M), rel
