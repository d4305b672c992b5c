"""C-ABI argument validation on CPU: invalid calls return the documented
status codes and reference-style messages before any CUDA work."""

import ctypes

import numpy as np
import pytest

from paper_1806_08422_b200 import _native

lib = _native.load()
ARG = _native.NMFA_ERR_ARG


def err():
    return lib.nmfa_last_error().decode()


def test_null_handles_are_rejected():
    out = ctypes.c_void_p()
    assert lib.nmfa_problem_create(5, 0, None, None, None, None, 0, None) == ARG
    assert lib.nmfa_plan_create(None, 4, 10, None, 0.15, 0.15, ctypes.byref(out)) == ARG
    assert lib.nmfa_plan_run(None, 0, 0, None, None, None, None, None, None, None, None) == ARG
    assert lib.nmfa_plan_run_sweeps(None, 0, 0, 0, 1, 0, None, None, None) == ARG
    assert lib.nmfa_plan_read_config(None, None, None) == ARG
    assert lib.nmfa_anneal_host(None, 4, 10, None, 0.15, 0.15, 0, 0, None, None) == ARG
    assert lib.nmfa_ground_state(None, 26, None, None, None) == ARG
    assert lib.nmfa_anneal_many(None, 0, 4, 10, None, 0.15, 0.15, None, None, None, None) == ARG
    assert lib.nmfa_best_of(None, 0, None, None, None) != 0
    assert lib.nmfa_problem_set_field_precision(None, 1) == ARG
    assert "NULL" in err()


def test_problem_validation_messages():
    out = ctypes.c_void_p()
    ei = np.array([0], np.int64)
    ej = np.array([0], np.int64)
    w = np.array([1.0])
    # the reference's IsingProblem errors (problem.py:25-62)
    assert lib.nmfa_problem_create(0, 0, None, None, None, None, 0, ctypes.byref(out)) == ARG
    assert "positive" in err()
    assert lib.nmfa_problem_create(3, 1, _native.ptr(ei), _native.ptr(ej), _native.ptr(w), None, 0,
                                   ctypes.byref(out)) == ARG
    assert "self" in err().lower()
    ej2 = np.array([7], np.int64)
    assert lib.nmfa_problem_create(3, 1, _native.ptr(ei), _native.ptr(ej2), _native.ptr(w), None, 0,
                                   ctypes.byref(out)) == ARG
    assert "range" in err()


def test_sk_device_shard_validation():
    out = ctypes.c_void_p()
    assert lib.nmfa_problem_create_sk_device(1, 0, 0, 1, 0, ctypes.byref(out)) == ARG
    assert lib.nmfa_problem_create_sk_device(1024, 0, 100, 600, 0, ctypes.byref(out)) == ARG
    assert "multiples of 128" in err()
    assert lib.nmfa_problem_create_sk_device(1024, 0, 512, 256, 0, ctypes.byref(out)) == ARG


def test_gset_parse_header_query_without_arrays():
    n, m = ctypes.c_int64(), ctypes.c_int64()
    text = b"5 2\n1 2 1\n3 4 -1\n"
    assert lib.nmfa_gset_parse(text, len(text), ctypes.byref(n), ctypes.byref(m), None, None,
                               None, 0) == 0
    assert (n.value, m.value) == (5, 2)
    ei = np.empty(1, np.int64)
    assert lib.nmfa_gset_parse(text, len(text), ctypes.byref(n), ctypes.byref(m),
                               _native.ptr(ei), _native.ptr(ei), _native.ptr(np.empty(1)), 1) == ARG
    assert "fewer than the declared" in err()


def test_version_and_errors_are_strings():
    assert b"sm_100a" in lib.nmfa_version()
    lib.nmfa_plan_destroy(None)
    assert isinstance(lib.nmfa_last_error(), bytes)


def test_round2_entry_points_validate_before_cuda():
    out = ctypes.c_void_p()
    buf = np.zeros(16, np.float32)
    # nmfa_reference_noise (the replay mode's device stream)
    assert lib.nmfa_reference_noise(0, 0, 0, 10, 0.15, _native.ptr(buf), None, None) == ARG
    assert "positive" in err()
    assert lib.nmfa_reference_noise(0, 0, 4, 10, 0.15, None, None, None) == ARG
    assert "no output buffer" in err()
    assert lib.nmfa_reference_noise(0, 0, 4, 10, -1.0, _native.ptr(buf), None, None) == ARG
    # nmfa_problem_create_bits_device (the bit-packed device format)
    bits = np.zeros(8, np.uint32)
    assert lib.nmfa_problem_create_bits_device(16, None, None, 0, 16, 0, ctypes.byref(out)) == ARG
    assert lib.nmfa_problem_create_bits_device(1, _native.ptr(bits), None, 0, 1, 0,
                                               ctypes.byref(out)) == ARG
    assert "n >= 2" in err()
    assert lib.nmfa_problem_create_bits_device(16, _native.ptr(bits), None, 8, 16, 0,
                                               ctypes.byref(out)) == ARG
    assert "multiples of 128" in err()
    assert lib.nmfa_problem_create_bits_device(16, _native.ptr(bits), None, 0, 17, 0,
                                               ctypes.byref(out)) == ARG
    h = np.full(16, np.inf)
    assert lib.nmfa_problem_create_bits_device(16, _native.ptr(bits), _native.ptr(h), 0, 16, 0,
                                               ctypes.byref(out)) == ARG
    assert "finite" in err()
    # nmfa_problem_create_gset: parse errors carry the reference's line numbers
    bad = b"3 2\n1 2 1\n1 9 1\n"
    assert lib.nmfa_problem_create_gset(bad, len(bad), 0, ctypes.byref(out)) == ARG
    assert err().startswith("line 3")
    assert lib.nmfa_problem_create_gset(None, 0, 0, ctypes.byref(out)) == ARG
    # the product library reports that it has no guard allocator
    assert lib.nmfa_debug_guard_check() == -1
