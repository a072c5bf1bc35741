"""The C-ABI library loads and exports every symbol include/voltana.h declares; host-side
validation rejects bad arguments synchronously (no GPU needed: nothing is enqueued)."""

import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def vt():
    import paper_2509_04827_b200 as vt
    from paper_2509_04827_b200 import build
    build.build()
    return vt


def declared_functions():
    src = open(os.path.join(ROOT, "include", "voltana.h")).read()
    return sorted(set(re.findall(r"\b(voltana_[a-z_]+)\s*\(", src)))


def test_header_symbols_exported(vt):
    names = declared_functions()
    assert len(names) >= 9
    L = vt.lib()
    for n in names:
        assert hasattr(L, n), n
    assert sorted(vt.exported_symbols()) == sorted(set(vt._lib.EXPORTS))


def test_status_strings(vt):
    L = vt.lib()
    assert L.voltana_status_string(0) == b"ok"
    assert L.voltana_status_string(6) == b"workspace too small"


def _profile(vt, k=3, tiles=1):
    p = vt._lib.Profile()
    p.k, p.n_tiles, p.tile_w = k, tiles, 128
    for f in ("mhz", "a1", "c1", "a2", "b2", "c2", "dyn"):
        setattr(p, f, 0x1000)  # never dereferenced: validation fails first
    p.p_idle, p.tdp, p.u_half_prefill, p.u_half_decode = 60.0, 400.0, 1024.0, 64.0
    return p


def test_host_validation_errors(vt):
    L = vt.lib()
    p = _profile(vt)
    bad = np.array([2, 1], np.uint16)
    rc = L.voltana_control_step(C.byref(p), 0, 0, bad.ctypes.data, 2, 1, 1, 1, 1, 1, 10, 1, 1, None)
    assert rc == 2 and b"strictly increasing" in L.voltana_last_error_detail()
    off = np.array([0, 5], np.uint16)
    rc = L.voltana_control_step(C.byref(p), 0, 0, off.ctypes.data, 2, 1, 1, 1, 1, 1, 10, 1, 1, None)
    assert rc == 3
    lad = np.array([0, 2], np.uint16)
    rc = L.voltana_control_step(C.byref(p), 7, 0, lad.ctypes.data, 2, 1, 1, 1, 1, 1, 10, 1, 1, None)
    assert rc == 1
    rc = L.voltana_control_step(C.byref(p), 1, 2, lad.ctypes.data, 2, 1, 1, 1, 1, 1, 10, 1, 1, None)
    assert rc == 1 and b"mode" in L.voltana_last_error_detail()                    # mode outside 0..1
    rc = L.voltana_route_batch(C.byref(p), lad.ctypes.data, 2, 2, 1, 1, 1, 1, 150, 3, 1, 10, 1, 1, 1, None)
    assert rc == 1 and b"policy" in L.voltana_last_error_detail()                  # policy outside 0..2
    lad = np.array([0, 2], np.uint16)
    rc = L.voltana_route_batch(C.byref(p), lad.ctypes.data, 2, 9, 1, 1, 1, 1, 150, 0, 1, 10, 1, 1, 1, None)
    assert rc == 5
    rc = L.voltana_fit_profile(1, 1, 1, 1, 1, 1, 100, 0, 1, 128, 0.0, 1, 2000, 1, 1, 1, 1, 1, 1, 1, None, None, 0, None)
    assert rc == 1
    rc = L.voltana_fit_profile(1, 1, 1, 1, 1, 1, 100, 3, 1, 128, 0.0, 1, 2000, 1, 1, 1, 1, 1, 1, 1, None, None, 0, None)
    assert rc == 6


def test_simulate_validation_errors(vt):
    L = vt.lib()
    lib = vt._lib
    tr = lib.Traces(1, 1, 1, 1, 1, 1, 10, 100, 0)
    slos = (lib.Slo * 1)(lib.Slo(600.0, 60.0, 1.0))
    lays = (lib.Layout * 1)(lib.Layout(2, 9, 0, 150, 8192, 400000, 0.0))
    g = lib.Grid(2)
    g.level[0], g.level[1] = 0, 1
    grids = (lib.Grid * 1)(g)
    profs = (lib.Profile * 1)(_profile(vt))
    sc = lib.Scenarios(1, 1, 1, 1, 1, 1)
    args = lambda lays, slos=slos, grids=grids: (C.byref(tr), slos, 1, lays, 1, grids, 1, profs, 1, C.byref(sc),
                                                 4, 1, 1, 0, None)
    assert L.voltana_simulate(*args(lays)) == 5                                     # N_D = 9
    lays[0].n_d = 2
    lays[0].kv_transfer_ms = 1e-5
    assert L.voltana_simulate(*args(lays)) == 5                                     # tau too small
    lays[0].kv_transfer_ms = 0.0
    assert L.voltana_simulate(*args(lays)) == 6                                     # no workspace
    lays[0].ctrl_mode = 2
    assert L.voltana_simulate(*args(lays)) == 5                                     # ctrl_mode outside 0..1
    lays[0].ctrl_mode = 0
    lays[0].policy = 3
    assert L.voltana_simulate(*args(lays)) == 5                                     # policy outside 0..2
    lays[0].policy = 0
    lays[0].ctrl_interval_ms = -1.0
    assert L.voltana_simulate(*args(lays)) == 5                                     # negative window
    lays[0].ctrl_interval_ms = 0.0
    lays[0].freq_overhead_ms = float("nan")
    assert L.voltana_simulate(*args(lays)) == 5                                     # NaN overhead
    lays[0].freq_overhead_ms = 0.0
    bad_slo = (lib.Slo * 1)(lib.Slo(-1.0, 60.0, 1.0))
    assert L.voltana_simulate(*args(lays, slos=bad_slo)) == 1
    g2 = lib.Grid(2)
    g2.level[0], g2.level[1] = 1, 1
    assert L.voltana_simulate(*args(lays, grids=(lib.Grid * 1)(g2))) == 2


def test_product_has_no_cpu_fallback():
    """The product package never imports the oracle or synth (parity evidence hygiene)."""
    pkg = os.path.join(ROOT, "paper_2509_04827_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f
                assert "oracle.h" not in src and "liboracle" not in src, f
                assert "import synth" not in src and "from synth" not in src, f


def test_simulate_workspace_grows_with_requests(vt):
    """K4 keeps one 16-B request node per request of every scenario (K4a -> K4b): n x
    max_requests x 16 B without node offsets, total_requests x 16 B with them; everything else
    is per resident warp (voltana.h, voltana_simulate_workspace_bytes[_ex])."""
    L = vt.lib()
    lib = vt._lib
    lays = (lib.Layout * 1)(lib.Layout(2, 2, 0, 150, 8192, 400000, 0.0))

    def ws(n, mr, total=None):
        tr = lib.Traces(1, 1, 1, 1, 1, 1, mr, 100, 0)
        if total is None:
            return int(L.voltana_simulate_workspace_bytes(C.byref(tr), lays, 1, n))
        return int(L.voltana_simulate_workspace_bytes_ex(C.byref(tr), lays, 1, n, total))

    assert ws(100, 2000) - ws(100, 1000) >= 100 * 1000 * 16
    assert ws(20000, 1000) - ws(10000, 1000) >= 10000 * 1000 * 16
    assert ws(4096, 45412) >= 4096 * 45412 * 16
    # node offsets: the node region is exactly 16 B per request of the sweep (to 256-B alignment)
    d = ws(4096, 45412, 90_000_000) - ws(4096, 45412, 80_000_000)
    assert abs(d - 10_000_000 * 16) <= 512
    assert ws(4096, 45412, 89_000_000) < ws(4096, 45412) - 4096 * 45412 * 16 + 89_000_000 * 16 + 1024
    assert ws(4096, 45412) == ws(4096, 45412, 0)


def test_fit_workspace_holds_the_warp_rows(vt):
    """K1 (one cooperative launch): the workspace holds a row block of cells x 5 doubles per
    resident warp (two CTAs of eight warps per SM bound the grid), the CTA partials and the grid
    sums; it does not depend on the sample count beyond that bound, and invalid shapes give 0."""
    L = vt.lib()
    k, T = 28, 16
    cells = k + T * k
    big = int(L.voltana_fit_workspace_bytes(10**8, k, T, 1))
    small = int(L.voltana_fit_workspace_bytes(1000, k, T, 1))
    rows_bound = 148 * 2 * 8 * cells * 5 * 8          # B200: 148 SMs
    assert big >= rows_bound
    assert big == int(L.voltana_fit_workspace_bytes(10**9, k, T, 1))   # bounded by the co-resident grid
    assert small == big                                  # partials and rows are sized for any grid
    assert int(L.voltana_fit_workspace_bytes(1000, 0, T, 1)) == 0
    assert int(L.voltana_fit_workspace_bytes(1000, k, 0, 1)) == 0
