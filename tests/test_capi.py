"""C-ABI boundary checks that run without a GPU.

* libgroot_b200.so loads and exports every function include/groot.h declares.
* Host-side entry points (CSA generator, AIGER parser, Glorot init) match the
  oracle bit for bit — they do not touch the device.
* Compute entry points fail loudly (GROOT_ECUDA) when no device is present:
  there is no CPU fallback.
"""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

from oracle import pyoracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _lib():
    from paper_2511_18297_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        from paper_2511_18297_b200 import build
        build.build()
    return _lib


def _declared():
    text = open(os.path.join(ROOT, "include", "groot.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(groot_[a-z0-9_]+)\s*\(", text)))


def test_header_declarations_are_exported():
    L = _lib()
    lib = L.lib()
    declared = _declared()
    assert len(declared) >= 50
    for name in declared:
        assert hasattr(lib, name), name
    assert sorted(L.EXPORTED) == declared
    out = subprocess.run(["nm", "-D", "--defined-only", L.LIB_PATH], capture_output=True, text=True).stdout
    for name in declared:
        assert re.search(rf"\bT {name}$", out, re.M), name


def test_library_is_sm100a():
    L = _lib()
    out = subprocess.run(["cuobjdump", "--list-elf", L.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", L.LIB_PATH], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass  # tcgen05.mma in the fused layer kernel
    assert "LDTM" in sass     # tcgen05.ld epilogue


@pytest.mark.parametrize("width", [2, 3, 4, 8, 17, 64])
def test_gen_csa_host_matches_oracle(width):
    from paper_2511_18297_b200 import api
    c = api.gen_csa_multiplier(width)
    o = O.gen_csa(width)
    assert c.aig.num_inputs == o.num_inputs
    np.testing.assert_array_equal(c.aig.and_lits, o.and_lits)
    np.testing.assert_array_equal(c.aig.out_lits, o.out_lits)
    np.testing.assert_array_equal(c.labels, o.labels)


def test_gen_csa_rejects_narrow():
    from paper_2511_18297_b200 import api
    with pytest.raises(ValueError, match="width must be >= 2"):
        api.gen_csa_multiplier(1)


def test_aiger_roundtrip_and_errors():
    from paper_2511_18297_b200 import api
    c = api.gen_csa_multiplier(8)
    text = api.write_aiger(c.aig)
    a = api.parse_aiger(text)
    np.testing.assert_array_equal(a.and_lits, c.aig.and_lits)
    np.testing.assert_array_equal(a.out_lits, c.aig.out_lits)
    cases = {
        "": "AIGER: empty input",
        "aig 1 1 0 0 0\n2\n": "expected ASCII header 'aag', got 'aig'",
        "aag 1 1 1 0 0\n2\n2 3\n": "latches unsupported",
        "aag 2 1 0 0 0\n2\n": r"non-contiguous variable numbering \(M != I \+ A\)",
        "aag 1 1 0 0 0\n4\n": "inputs must be the literals 2..2I in order",
        "aag 2 1 0 0 1\n2\n6 2 2\n": "AND definitions must appear in ascending index order",
        "aag 2 1 0 0 1\n2\n4 4 2\n": r"fanin index >= own index \(cycle\)",
        "aag 2 1 0 1 1\n2\n99\n4 2 2\n": "output literal out of range",
    }
    for text, msg in cases.items():
        with pytest.raises(RuntimeError, match=msg):
            api.parse_aiger(text)


def test_init_params_match_oracle():
    from paper_2511_18297_b200 import api
    for seed, depth in ((7, 4), (0, 3), (123, 1)):
        np.testing.assert_array_equal(api.init_params(seed, depth=depth), O.init_model(seed, depth=depth))
    assert api.param_count() == 6693


def test_asg1_golden_model_header(golden_dir):
    data = open(os.path.join(golden_dir, "trained_csa8.asg1"), "rb").read()
    assert data[:4] == b"ASG1"
    assert np.frombuffer(data[4:20], np.uint32).tolist() == [4, 4, 32, 5]
    assert len(data) == 20 + 8 * 6693


def test_compute_without_device_fails_loudly():
    """No CPU fallback: encode needs the device."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a device is present")
    from paper_2511_18297_b200 import api, GrootError
    c = api.gen_csa_multiplier(2)
    with pytest.raises(GrootError):
        api.encode(c.aig, c.labels)


def test_assignment_ids_beyond_n_are_rejected_before_sizing():
    """a part id >= n (e.g. -1 cast to u32) must not size the empty-part
    table by the id; the reference reports the first empty partition."""
    from paper_2511_18297_b200 import api
    for bad, first_empty in ((0xFFFFFFFF, 2), (7, 2), (3, 2)):
        part = np.array([0, 1, bad, 1], np.uint32)
        with pytest.raises(RuntimeError, match=f"assignment: empty partition {first_empty}$"):
            api.PartitionAssignment.from_host(part)


def test_parts_from_host_validation():
    from paper_2511_18297_b200 import api
    P = api.AugmentedPartition
    bad_core = [P(np.array([0, 9], np.uint32), np.zeros(0, np.uint32), np.zeros((0, 2), np.uint32))]
    with pytest.raises(ValueError, match="core node id out of range"):
        api.AugmentedPartitions.from_host(5, bad_core)
    bad_edge = [P(np.array([0, 1], np.uint32), np.array([2], np.uint32), np.array([[0, 3]], np.uint32))]
    with pytest.raises(ValueError, match="local edge endpoint out of range"):
        api.AugmentedPartitions.from_host(5, bad_edge)
