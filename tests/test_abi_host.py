"""CPU-side checks of the boundary: the C-ABI library loads, exports every
symbol include/rld.h declares, and its struct layouts agree with the ctypes
mirror; host-side API validation mirrors the reference's ValueErrors."""

import ctypes as C
import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT
from paper_2405_03474_b200 import _native as N
from paper_2405_03474_b200.estimators import EstimatorConfig, make_config
from paper_2405_03474_b200.kernels import KernelSpec, kernel_value
from paper_2405_03474_b200.linalg import Rng, philox_key
from paper_2405_03474_b200.parallel import shard_bounds
from paper_2405_03474_b200.precond import PreconditionerConfig

HEADER = ROOT / "include" / "rld.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^(?:int|void\*?|const char\*)\s+(rld_\w+)\(", text, re.M)))


def test_header_symbols_match_binding():
    assert declared_symbols() == sorted(N.EXPORTS)


def test_library_loads_and_exports_every_symbol():
    lib = N.load()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert lib.rld_abi_version() == N.ABI_VERSION == 4


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", str(N.LIB_PATH)], capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    assert "sm_100a" in out.stdout


C_PROBE = r"""
#include <stdio.h>
#include <stddef.h>
#include "rld.h"
#define P(T) printf(#T " %zu\n", sizeof(T));
#define O(T, f) printf(#T "." #f " %zu\n", offsetof(T, f));
int main(void) {
  P(rld_device_set) P(rld_problem) P(rld_config) P(rld_inputs) P(rld_result)
  O(rld_problem, data) O(rld_problem, ld) O(rld_config, probe_key) O(rld_config, omega_key)
  O(rld_config, diag_floor) O(rld_result, per_probe) O(rld_result, phase_ms) O(rld_inputs, memory)
  O(rld_config, estimator) O(rld_result, clamped_eigs) O(rld_config, precond_scale) O(rld_config, precond_key)
  O(rld_device_set, comm_kind) O(rld_device_set, nccl_id) O(rld_device_set, group)
  return 0;
}
"""


def test_struct_layouts_match_ctypes(tmp_path):
    src = tmp_path / "probe.c"
    src.write_text(C_PROBE)
    exe = tmp_path / "probe"
    r = subprocess.run(["gcc", "-I", str(ROOT / "include"), str(src), "-o", str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    got = dict(line.rsplit(" ", 1) for line in subprocess.check_output([str(exe)], text=True).splitlines())
    mirror = {"rld_device_set": N.DeviceSet, "rld_problem": N.Problem, "rld_config": N.Config,
              "rld_inputs": N.Inputs, "rld_result": N.Result}
    for cname, cls in mirror.items():
        assert int(got[cname]) == C.sizeof(cls), cname
    for key, val in got.items():
        if "." in key:
            cname, field = key.split(".")
            assert int(val) == getattr(mirror[cname], field).offset, key


def test_create_without_gpu_fails_cleanly():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError):
        N.Handle(0)


def test_config_validation_mirrors_reference():
    with pytest.raises(ValueError):
        EstimatorConfig(algorithm="r4")
    with pytest.raises(ValueError):
        EstimatorConfig(num_probes=0)
    with pytest.raises(ValueError):
        EstimatorConfig(lanczos_iters=0)
    with pytest.raises(ValueError):
        EstimatorConfig(dtype="bf16")
    with pytest.raises(ValueError):
        PreconditionerConfig(kind="nope")
    with pytest.raises(ValueError):
        PreconditionerConfig(rank=-1)
    with pytest.raises(ValueError):
        PreconditionerConfig(num_iters=0)
    with pytest.raises(ValueError):
        KernelSpec("cosine")
    with pytest.raises(ValueError):
        KernelSpec(length_scale=0.0)
    with pytest.raises(ValueError):
        make_config(EstimatorConfig(algorithm="exact"), 10)
    with pytest.raises(ValueError):
        make_config(EstimatorConfig(precond=PreconditionerConfig("partial-cholesky", 11)), 10)
    assert make_config(EstimatorConfig(precond=PreconditionerConfig("rank-one", 50)), 10).precond_kind == \
        N.PRECOND_RANK_ONE
    with pytest.raises(ValueError):
        make_config(EstimatorConfig(precond=PreconditionerConfig("trunc-svd", 11)), 10)


def test_make_config_fields():
    cfg = EstimatorConfig("r5", 16, 20, "rademacher", PreconditionerConfig("rand-svd", 64, 5), 7)
    c = make_config(cfg, 2048)
    assert (c.order, c.num_probes, c.lanczos_iters, c.precond_rank, c.precond_iters, c.oversample) == \
        (5, 16, 20, 64, 5, 10)
    assert (c.probe_key[0], c.probe_key[1]) == philox_key(7, (2,))
    assert (c.omega_key[2], c.omega_key[3]) == philox_key(7, (1, 1))


def test_make_config_slq_runs_without_preconditioner():
    # src/estimators.py:106: SLQ ignores the preconditioner config
    c = make_config(EstimatorConfig("slq", 8, 20, precond=PreconditionerConfig("partial-cholesky", 5)), 100)
    assert c.estimator == N.ESTIMATOR_SLQ and c.precond_kind == N.PRECOND_IDENTITY
    assert make_config(EstimatorConfig("r3"), 100).estimator == N.ESTIMATOR_RSTAR


def test_philox_key_is_numpy_state():
    st = np.random.Philox(np.random.SeedSequence(3, spawn_key=(2,))).state["state"]
    assert philox_key(3, (2,)) == tuple(int(k) for k in st["key"])


def test_rng_facade_matches_reference_streams(golden_streams):
    np.testing.assert_array_equal(Rng(0).child(2).rademacher((3, 37)), golden_streams["rademacher_seed0"])


def test_kernel_value_known_answers(golden_units):
    assert kernel_value(KernelSpec("rbf"), [0.0], [1.0]) == pytest.approx(golden_units["kernel_r1_rbf"], rel=1e-15)
    assert kernel_value(KernelSpec("matern52"), [0.0], [1.0]) == pytest.approx(golden_units["kernel_r1_matern52"],
                                                                               rel=1e-15)


def test_shard_bounds_cover_rows():
    for n in (1, 7, 2048, 65537):
        for world in (1, 2, 3, 8):
            spans = [shard_bounds(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c and a <= b


def _words_consumed(bg):
    st = bg.state
    ctr = int(st["state"]["counter"][0])
    return 0 if ctr == 0 else 4 * (ctr - 1) + int(st["buffer_pos"])


@pytest.mark.parametrize("seed,path,k,df,m", [(0, (2, 0), 4096 * 3, 4096, 3), (7, (2, 1), 12345, 12345, 8),
                                              (3, (2, 0), 100, 5, 50), (11, (1,), 0, 1000, 4)])
def test_host_chi_radii_continue_numpy_stream(seed, path, k, df, m):
    """rld_chi_radii (host port of numpy's chisquare) continues the Philox stream where
    the device's Gaussian rows stopped: bit-identical to Generator.chisquare (src/linalg.py:87-88)."""
    g = np.random.Generator(np.random.Philox(np.random.SeedSequence(seed, spawn_key=path)))
    g.standard_normal(k)
    w0 = _words_consumed(g.bit_generator)
    want = np.sqrt(g.chisquare(df, m))
    lib = N.load()
    key = (C.c_uint64 * 2)(*philox_key(seed, path))
    out = np.empty(m)
    assert lib.rld_chi_radii(C.byref(key), w0, df, m, out.ctypes.data) == 0
    np.testing.assert_array_equal(out, want)
