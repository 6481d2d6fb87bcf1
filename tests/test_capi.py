"""CPU-side checks of the C ABI boundary: the library loads without a GPU and
exports exactly what include/hexamoe.h declares; host-only entry points
(input generators) reproduce the reference's seeded streams."""
import os
import re

import numpy as np
import pytest

import oracle as O
from paper_2411_01288_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "hexamoe.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hxm_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    names = declared_symbols()
    assert len(names) >= 18
    for n in names:
        assert hasattr(L, n), n
    # and the ctypes table covers the whole header
    assert set(names) == set(_lib.SIGNATURES), set(names) ^ set(_lib.SIGNATURES)


def test_host_checks_precede_device_work():
    L = _lib.lib()
    # blk == 0 is rejected before any launch (routing.cpp:44)
    assert L.hxm_build_reindex(None, 4, 2, 0, None, None, None, 0, None, None) == 2
    assert L.hxm_reindex_bound(5, 2, 2) == 7
    assert L.hxm_version() >= 100


def test_synthesize_routing_matches_reference_stream():
    from paper_2411_01288_b200 import synthesize_routing
    for dist in ("uniform", "zipf:1.2", "fixed:2", "balanced"):
        r = synthesize_routing(257, 7, 3, dist, 11)
        assert np.array_equal(r.assignments, O.synthesize_routing(257, 7, 3, dist, 11))
        r.validate()
    with pytest.raises(ValueError):
        synthesize_routing(4, 2, 3)


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_layer_inputs_match_reference_generator():
    import ctypes as C
    E, din, hid, dout, n = 3, 5, 7, 4, 9
    x, w1, b1, w2, b2 = O.ref_make_inputs(42, E, din, hid, dout, n)
    bufs = [np.empty(a.shape, np.float32) for a in (w1, b1, w2, b2, x)]
    _lib.lib().hxm_make_layer_inputs(42, E, din, hid, dout, n, 0.5,
                                     *[b.ctypes.data for b in bufs])
    for got, want in zip(bufs, (w1, b1, w2, b2, x)):
        assert np.array_equal(got, want.astype(np.float32))


def test_routing_csv_round_trip():
    from paper_2411_01288_b200 import routing_from_csv, routing_to_csv, synthesize_routing
    r = synthesize_routing(17, 5, 2, "uniform", 3)  # test_routing.cpp:149-162
    back = routing_from_csv(routing_to_csv(r))
    assert np.array_equal(back.assignments, r.assignments)
    with pytest.raises(ValueError):
        routing_from_csv("token_index,choice_index,expert_id\n0,0,1\n2,0,0\n")
    with pytest.raises(ValueError):
        routing_from_csv("")
