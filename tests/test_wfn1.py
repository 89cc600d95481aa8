"""WFN1 orbital files (reference model.hpp:236-339): the
product reader / writer (liblrgw_cuda.so, paper_2403_12340_b200/csrc/wfn1.cpp)
against the reference's own save_system / load_system (oracle/_ref): identical
bytes, cross-readable files, the same io_error cases and messages
(test_model.cpp:125-193). Host I/O only — runs without a GPU."""
import ctypes
import os

import numpy as np
import pytest

from paper_2403_12340_b200 import lrgw

CELLS = [(6.0, 6.0, 6.0), (10.26, 10.26, 10.26), (20.52, 30.78, 41.04), (0.75, 1e-5, 123456.789),
         (1.0 / 3.0, 2.5e17, 7e-7)]


def _system(dims, cell, n_v, n_c, seed=0):
    rng = np.random.default_rng(seed)
    n_r = int(np.prod(dims))
    return lrgw.ElectronicStructure(tuple(dims), tuple(cell), np.asfortranarray(rng.standard_normal((n_r, n_v + n_c))),
                                    np.sort(rng.uniform(-1, 1, n_v + n_c)), rng.uniform(-0.1, 0.1, n_v + n_c),
                                    n_v, n_c)


def _ref_message(ref, path):
    lib = ref.lib()
    lib.ref_last_message.restype = ctypes.c_char_p
    d = np.zeros(3, dtype=np.int32)
    c = np.zeros(3)
    nv, nc = ctypes.c_int(0), ctypes.c_int(0)
    rc = lib.ref_load_system(str(path).encode(), d.ctypes.data_as(ctypes.POINTER(ctypes.c_int)),
                             c.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), ctypes.byref(nv), ctypes.byref(nc),
                             None, None, None)
    return rc, lib.ref_last_message().decode()


@pytest.mark.parametrize("cell", CELLS)
def test_writer_bytes_match_reference(ref, tmp_path, cell):
    es = _system((4, 4, 2), cell, 2, 3)
    ours, theirs = tmp_path / "ours.wfn1", tmp_path / "ref.wfn1"
    lrgw.save_system(ours, es)
    ref.save_system(theirs, es.dims, es.cell, es.n_v, es.n_c, es.psi, es.energies, es.vxc)
    assert ours.read_bytes() == theirs.read_bytes()


def test_round_trip_and_cross_read(ref, tmp_path):
    es = _system((6, 4, 4), (5.0, 6.5, 7.25), 3, 5, seed=2)
    p = tmp_path / "a.wfn1"
    lrgw.save_system(p, es)
    back = lrgw.load_system(p)
    assert back.dims == es.dims and back.cell == es.cell and (back.n_v, back.n_c) == (3, 5)
    assert np.array_equal(back.psi, es.psi)
    assert np.array_equal(back.energies, es.energies) and np.array_equal(back.vxc, es.vxc)
    dims, cell, nv, nc, psi, e, v = ref.load_system(p)  # the reference reads ours
    assert (dims, cell, nv, nc) == (es.dims, es.cell, 3, 5) and np.array_equal(psi, es.psi)
    q = tmp_path / "b.wfn1"
    ref.save_system(q, es.dims, es.cell, 3, 5, es.psi, es.energies, es.vxc)  # we read the reference's
    back = lrgw.load_system(q)
    assert np.array_equal(back.psi, es.psi) and np.array_equal(back.vxc, es.vxc)


def _header_file(path, header: bytes, payload: bytes = b"", magic=b"WFN1"):
    with open(path, "wb") as f:
        f.write(magic + len(header).to_bytes(4, "little") + header + payload)


CORRUPT = {
    # name -> (writer, exact-message?)
    "bad_magic": (lambda p, good: p.write_bytes(b"XFN1" + good[4:]), True),
    "short_magic": (lambda p, good: p.write_bytes(b"WF"), True),
    "no_length": (lambda p, good: p.write_bytes(b"WFN1\x10\x00"), True),
    "short_header": (lambda p, good: p.write_bytes(good[:12]), True),
    "truncated_psi": (lambda p, good: p.write_bytes(good[:-(8 * 16 + 8)]), True),
    "truncated_vxc": (lambda p, good: p.write_bytes(good[:-4]), True),
    "nr_mismatch": (lambda p, good: _header_file(p, b'{"dims":[4,4,2],"cell":[5.0,5.0,5.0],"nr":33,"nv":2,"nc":2}'),
                    True),
    "bands": (lambda p, good: _header_file(p, b'{"dims":[2,2,2],"cell":[5.0,5.0,5.0],"nr":8,"nv":0,"nc":2}'), True),
    "bands_big": (lambda p, good: _header_file(p, b'{"dims":[2,2,2],"cell":[5,5,5],"nr":8,"nv":5,"nc":4}'), True),
    "grid": (lambda p, good: _header_file(p, b'{"dims":[1,4,4],"cell":[5.0,5.0,5.0],"nr":16,"nv":1,"nc":1}'), False),
    "cell": (lambda p, good: _header_file(p, b'{"dims":[2,4,4],"cell":[5.0,0,5.0],"nr":32,"nv":1,"nc":1}'), False),
    "json": (lambda p, good: _header_file(p, b'{"dims":[4,4,2],"cell":[5.0,5.0'), False),
    "missing_key": (lambda p, good: _header_file(p, b'{"dims":[4,4,2],"cell":[5.0,5.0,5.0],"nv":2,"nc":2}'), False),
    "wrong_type": (lambda p, good: _header_file(p, b'{"dims":"444","cell":[5.0,5.0,5.0],"nr":32,"nv":2,"nc":2}'),
                   False),
    "short_dims": (lambda p, good: _header_file(p, b'{"dims":[4,4],"cell":[5.0,5.0,5.0],"nr":16,"nv":2,"nc":2}'),
                   False),
}


@pytest.mark.parametrize("name", sorted(CORRUPT))
def test_corrupt_files_raise_like_reference(ref, tmp_path, name):
    es = _system((4, 2, 2), (5.0, 5.0, 5.0), 2, 2)
    good = tmp_path / "good.wfn1"
    lrgw.save_system(good, es)
    bad = tmp_path / f"{name}.wfn1"
    writer, exact = CORRUPT[name]
    writer(bad, good.read_bytes())
    rc, want = _ref_message(ref, bad)
    assert rc != 0, "the reference accepts this file"
    with pytest.raises(lrgw.IoError) as ei:
        lrgw.load_system(bad)
    got = str(ei.value)
    if exact:
        assert got == want
    else:  # nlohmann's exception text follows the reference's prefix
        prefix = want.split(": ")[0] + ": " + want.split(": ")[1]
        assert got.startswith(prefix), (got, want)


def test_missing_file_and_unwritable(ref, tmp_path):
    with pytest.raises(lrgw.IoError) as ei:
        lrgw.load_system(tmp_path / "lrgw_test_does_not_exist.wfn1")
    assert str(ei.value).startswith("load_system: cannot open")
    with pytest.raises(lrgw.IoError):
        lrgw.save_system(tmp_path / "no_dir" / "x.wfn1", _system((2, 2, 2), (1.0, 1.0, 1.0), 1, 1))


def test_header_variants_accepted_like_reference(ref, tmp_path):
    """Whitespace, key order, integral cells and extra keys are read the same."""
    n_r, nb = 8, 3
    rng = np.random.default_rng(5)
    payload = rng.standard_normal(n_r * nb + 2 * nb).tobytes()
    p = tmp_path / "v.wfn1"
    _header_file(p, b' { "nv" : 1, "nc":2, "nr":8, "cell":[3,4,5.5], "dims":[2,2,2], "extra":{"a":[true,null]} } ',
                 payload)
    back = lrgw.load_system(p)
    dims, cell, nv, nc, psi, e, v = ref.load_system(p)
    assert back.dims == dims and back.cell == cell and (back.n_v, back.n_c) == (nv, nc)
    assert np.array_equal(back.psi, psi) and np.array_equal(back.energies, e) and np.array_equal(back.vxc, v)
