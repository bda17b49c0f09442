"""Run-to-run determinism of every GPU stage (the reference is deterministic:
tests/test_assembly.py:204-210 bit-identical assembly, tests/test_acceptance.py:
316-328 byte-identical sweep CSVs).  No kernel uses atomics for values; every
reduction has a fixed order, so repeated calls — and the same frequencies in
different batches or concurrent streams — must agree bit for bit.  This is
also the harness that would expose a timing-dependent race (round 1 found one
in vb_zgetrs by chance)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _same(a, b):
    import torch
    return torch.equal(a, b) if isinstance(a, torch.Tensor) else np.array_equal(a, b)


@pytest.mark.parametrize("r", [48, 300, 1024])
def test_sweep_repeat_split_and_concurrent_streams(cuda, r):
    import torch
    from paper_2310_04734_b200 import sweep, workloads
    w = workloads.cfg5(r=r, n_freq=301)
    rs = sweep.ReducedSweep(w.prims, w.b, w.c_r, kinds=w.kinds)
    f = torch.as_tensor(w.freqs, device=cuda)
    a, b = rs.sweep_device(f), rs.sweep_device(f)
    assert _same(a.y, b.y) and _same(a.spl, b.spl)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    r1 = sweep.ReducedSweep(w.prims, w.b, w.c_r, kinds=w.kinds, stream=s1)
    r2 = sweep.ReducedSweep(w.prims, w.b, w.c_r, kinds=w.kinds, stream=s2)
    c1, c2 = r1.sweep_device(f[:151]), r2.sweep_device(f[151:])
    torch.cuda.synchronize()
    assert _same(c1.y, a.y[:151]) and _same(c2.y, a.y[151:])
    assert _same(c1.spl, a.spl[:151]) and _same(c2.spl, a.spl[151:])


def test_offline_stages_repeat_bit_identical(cuda):
    """FOM factor + solve (dense LU, FDM, GMRES), Krylov blocks, both
    orthonormalisation paths, projection (SpMM + split-K GEMM), twice each."""
    import torch
    from paper_2310_04734_b200 import linalg, mor, workloads
    fom, lay = workloads.cfg1_model(box=(0, 0, 0, 1.0, 0.8, 0.6), ne=(4, 3, 3), n_rec=6)
    runs = []
    for _ in range(2):
        Q, _ = mor.krylov_block_dev(fom, 140.0, 4, second_order=True)
        V = mor._orthonormalise(None, Q)
        rom = mor.ReducedModel(fom=fom, V=V, window=(20.0, 300.0))
        P, _, br = rom._projected()
        y, spl, _, _ = rom.sweep([30.0, 111.0, 290.0])
        runs.append((Q, V, P, br, y, spl))
    for x1, x2 in zip(*runs):
        assert _same(x1, x2)
    fom3, _ = workloads.cfg3_model(box=(0, 0, 0, 1.2, 0.6, 0.5), ne=(8, 4, 4), per_element_z=True)
    b = fom3.load_dev(120.0)
    g1 = fom3.factor(120.0).solve(b)
    g2 = fom3.factor(120.0).solve(b)
    assert _same(g1, g2)
    blocks = [Q for Q, _ in mor.krylov_blocks_mimo_dev(fom3, 120.0, 3, second_order=True)]
    Va = mor.orthonormalise_blocks(None, [q.clone() for q in blocks])
    Vb = mor.orthonormalise_blocks(None, [q.clone() for q in blocks])
    assert _same(Va, Vb)
    fom4, _ = workloads.cfg3_model(box=(0, 0, 0, 1.2, 0.6, 0.5), ne=(8, 4, 4))
    f1 = fom4.factor(77.0).solve(fom4.load_dev(77.0))
    f2 = fom4.factor(77.0).solve(fom4.load_dev(77.0))
    assert _same(f1, f2)
    Kg = lay["Kg"]
    X = torch.randn(Kg.n, 40, dtype=torch.complex128, device=cuda)
    for path in ("csr", "rg"):
        assert _same(linalg.spmm(Kg, X, path=path), linalg.spmm(Kg, X, path=path))
    W = torch.randn(Kg.n, 40, dtype=torch.complex128, device=cuda)
    assert _same(linalg.zgemm("C", X, W), linalg.zgemm("C", X, W))


def test_cfg4_assembly_and_plane_solver_repeat_bit_identical(cuda):
    """cfg4: facet-shell / chain-rule element kernels + CSR gather, and the
    plane-block factor + solve (LUs, block inverses, SpMM Schur updates,
    batched GEMVs), twice each."""
    from paper_2310_04734_b200 import fuselage as fz
    spec = fz.FuselageSpec(n_th=16, n_stringers=8, n_z=6, floor_k=1, n_side=2)
    fa, ia = fz.fuselage_model(spec, cuda)
    fb, ib = fz.fuselage_model(spec, cuda)
    for name in ("Ks", "Ms", "Kc", "Mi", "Cs", "CTi"):
        assert _same(ia[name].data, ib[name].data) and _same(ia[name].indices, ib[name].indices), name
    x = [fa.factor(173.0).solve(fa.load_dev(173.0)) for _ in range(2)]
    assert _same(x[0], x[1])
