"""Drop-in for the reference's assembled model: a `vibrofem.assembly.ModelOperator`
(assembly.py:221-287) read as DATA and turned into the GPU-native affine
operator, so `fom_from_operator(op, probe)` (mor.py:397-402) runs the whole MOR
path on the device without ever densifying an n x n matrix.

Why this is exact: every frequency dependence of the reference's operator is a
complex scalar in front of a frequency-independent sparse primitive
(assembly.py:242-257 per domain, 193-207 / 262-265 per coupling):

  elastic domain d      K += s_d(f) Kmat_d + Kgeo_d        M += M_d
  acoustic / JCA fluid  K += s_d(f) / rho_d(f) Kgrad_d     M += Mnn_d / (rho_d(f) c_d(f)^2)
  coupling (s, f, C)    K[s rows, f cols] += -C            M[f rows, s cols] += rho_f(f) C^T

with s_d = materials.complex_stiffness_scale (1 + i eta(f)), (rho_d, c_d) =
materials.jca_effective for an equivalent fluid, rho_f = assembly.fluid_density.
The primitives are embedded at their block offsets (op.block_map) as real
device CSR matrices; the scalars are host callables.  By default they are the
reference's own functions, resolved from the operator's module (the drop-in
runs inside the reference process; the product never imports `vibrofem`), or
they can be given explicitly (`OperatorCoefficients`), e.g. from tabulated
values.  The load stays the reference provider op.load(f) (plane_wave_load,
assembly.py:108-139), evaluated on the host and uploaded as one block per
batch of frequencies.
"""

from __future__ import annotations

import sys
import types
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp
import torch

from .assembly import DeviceCSR
from .mor import AffineOperator, AffineTerm

CDT = torch.complex128


def _embed(A, row_off: int, col_off: int, n: int) -> sp.csr_matrix:
    """A (rows x cols, any scipy format) placed at (row_off, col_off) of an
    n x n matrix; canonical CSR (sorted indices, duplicates summed, explicit
    zeros kept — scipy's coo -> csr, assembly.py:172-173)."""
    C = sp.coo_matrix(A)
    out = sp.coo_matrix((C.data, (C.row + row_off, C.col + col_off)), shape=(n, n)).tocsr()
    out.sum_duplicates()
    out.sort_indices()
    return out


def device_csr_terms(A, device, row_off: int = 0, col_off: int = 0, n: int | None = None):
    """[(DeviceCSR, complex factor)] with sum_k factor_k P_k = A embedded at
    (row_off, col_off): a real matrix is one term, a complex one two real terms
    (real part, imaginary part x 1j) on the same pattern."""
    n = n or A.shape[0]
    S = _embed(A, row_off, col_off, n)
    ip = torch.as_tensor(S.indptr.astype(np.int32), device=device)
    ix = torch.as_tensor(S.indices.astype(np.int32), device=device)
    d = S.data
    terms = [(DeviceCSR(n, ip, ix, torch.as_tensor(np.ascontiguousarray(d.real, dtype=np.float64),
                                                     device=device)), 1.0 + 0j)]
    if np.iscomplexobj(d) and np.any(d.imag != 0):
        terms.append((DeviceCSR(n, ip, ix, torch.as_tensor(np.ascontiguousarray(d.imag), device=device)), 1j))
    return terms


@dataclass
class OperatorCoefficients:
    """Per-frequency scalars of a ModelOperator (assembly.py:242-265):
    kscale(domain_id, f) -> complex stiffness scale (1 + i eta(f));
    fluid(domain_id, f) -> (rho_eff, c_eff) of a fluid domain;
    rho_f(coupling_index, f) -> density of the coupling's fluid side."""

    kscale: object
    fluid: object
    rho_f: object


def reference_coefficients(op) -> OperatorCoefficients:
    """The reference's own scalar functions (materials.complex_stiffness_scale,
    materials.jca_effective, assembly.fluid_density), found through the
    operator's module — the same calls _domain_KM / system make."""
    mod = sys.modules[type(op).__module__]
    mats, fluid_density = mod.mats, mod.fluid_density
    cfg = op.config
    doms = {d.id: d for d in cfg.domains}

    def kscale(did, f):
        table = cfg.damping_tables.get(doms[did].damping_table_id)
        return complex(mats.complex_stiffness_scale(table, f)) if table else 1.0 + 0j

    def fluid(did, f):
        d = doms[did]
        mat = cfg.materials[d.material_id]
        if d.kind == "equivalent_fluid":
            rho, c = mats.jca_effective(mat, f)
            return complex(rho), complex(c)
        return complex(mat.rho), complex(mat.c)

    def rho_f(k, f):
        sid, fid, _ = op.couplings[k]
        return complex(fluid_density(op.kinds[fid], cfg.material_of(fid), f))

    return OperatorCoefficients(kscale, fluid, rho_f)


class HostLoad:
    """The reference's load provider f -> ndarray(n) (host), with the device
    views the GPU path uses: at(f) (n x 1) and batch(freqs) (n x F, one upload
    per batch of frequencies)."""

    def __init__(self, fn, n: int, device):
        self.fn, self.n, self.device = fn, n, torch.device(device)

    def host(self, f):
        return np.asarray(self.fn(f))

    def at(self, f) -> torch.Tensor:
        return torch.as_tensor(np.asarray(self.fn(f), dtype=complex)).view(-1, 1).to(self.device)

    def batch(self, freqs) -> torch.Tensor:
        B = np.stack([np.asarray(self.fn(float(f)), dtype=complex) for f in freqs], axis=1)
        return torch.from_numpy(np.ascontiguousarray(B)).pin_memory().to(self.device, non_blocking=True)


def affine_from_operator(op, coeffs: OperatorCoefficients | None = None, device=None,
                         load=None) -> AffineOperator:
    """AffineOperator (device CSR primitives x host scalars) equal to the
    reference operator: K(f), M(f) of ModelOperator.system(f).assemble_K/M
    (assembly.py:193-218, 259-284) term by term.  Reads op.config.domains,
    op.kinds, op.block_map, op.primitives and op.couplings only."""
    dev = torch.device(device or "cuda")
    coeffs = coeffs or reference_coefficients(op)
    n = int(sum(size for _, size in op.block_map.values()))
    K, M = [], []

    def add(lst, A, off_r, off_c, coeff):
        for P, fac in device_csr_terms(A, dev, off_r, off_c, n):
            if callable(coeff):
                lst.append(AffineTerm(P, (lambda f, c=coeff, fac=fac: fac * c(f))))
            else:
                lst.append(AffineTerm(P, fac * complex(coeff)))

    for d in op.config.domains:
        off, _ = op.block_map[d.id]
        prim = op.primitives[d.id]
        if d.kind == "elastic":
            add(K, prim["Kmat"], off, off, lambda f, i=d.id: coeffs.kscale(i, f))
            add(K, prim["Kgeo"], off, off, 1.0)
            add(M, prim["M"], off, off, 1.0)
        else:
            def kcoef(f, i=d.id):
                rho, _ = coeffs.fluid(i, f)
                return coeffs.kscale(i, f) / rho

            def mcoef(f, i=d.id):
                rho, c = coeffs.fluid(i, f)
                return 1.0 / (rho * c * c)
            add(K, prim["Kgrad"], off, off, kcoef)
            add(M, prim["Mnn"], off, off, mcoef)
    for k, (sid, fid, C) in enumerate(op.couplings):
        so, _ = op.block_map[sid]
        fo, _ = op.block_map[fid]
        add(K, -sp.csr_matrix(C), so, fo, 1.0)                                  # -C on structure rows
        add(M, sp.csr_matrix(C).T, fo, so, lambda f, k=k: coeffs.rho_f(k, f))   # rho_f C^T on fluid rows
    ld = load if load is not None else HostLoad(op.load, n, dev)
    return AffineOperator(K=K, M=M, D=[], load=ld)


def load_operator_npz(path, device=None):
    """A reference model shipped as arrays (the layout
    tests/golden/make_fuselage_golden.py writes from a live ModelOperator:
    primitives, couplings, block map, the per-frequency scalars tabulated on a
    grid, the load's nonzero rows) -> (FullOrderModel on the device, grid,
    data).  Lets the drop-in run a reference model on a machine without the
    reference package; the scalars are looked up at the tabulated
    frequencies only."""
    from .mor import fom_from_operator
    with np.load(path) as zf:   # materialised: the coefficient callables run on several host threads
        z = {k: zf[k] for k in zf.files}
    grid = z["grid"]
    pos = {float(f): i for i, f in enumerate(grid)}
    doms = [str(d) for d in z["domains"]]
    kinds = {d: str(k) for d, k in zip(doms, z["kinds"])}

    def csr(key):
        return sp.csr_matrix((z[f"{key}__data"], z[f"{key}__indices"], z[f"{key}__indptr"]),
                             shape=tuple(z[f"{key}__shape"]))
    prims = {d: {nm: csr(f"prim__{d}__{nm}")
                 for nm in (("Kmat", "Kgeo", "M") if kinds[d] == "elastic" else ("Kgrad", "Mnn"))}
             for d in doms}
    couplings = [(str(a), str(b), csr(f"coupling{k}")) for k, (a, b) in enumerate(z["couplings"])]
    block_map = {d: tuple(int(v) for v in z["block_map"][i]) for i, d in enumerate(doms)}
    cfg = types.SimpleNamespace(domains=[types.SimpleNamespace(id=d, kind=kinds[d]) for d in doms])
    op = types.SimpleNamespace(config=cfg, kinds=kinds, primitives=prims, couplings=couplings,
                               block_map=block_map)
    coeffs = OperatorCoefficients(
        kscale=lambda d, f: complex(z[f"scale__{d}"][pos[float(f)]]),
        fluid=lambda d, f: (complex(z[f"rho_eff__{d}"][pos[float(f)]]), complex(z[f"c_eff__{d}"][pos[float(f)]])),
        rho_f=lambda k, f: complex(z[f"rho_f{k}"][pos[float(f)]]))
    n = int(z["n"])
    rows, vals = z["load_rows"], z["load_vals"]

    def load(f):
        v = np.zeros(n, complex)
        v[rows] = vals[pos[float(f)]]
        return v
    dev = torch.device(device or "cuda")
    op.affine = affine_from_operator(op, coeffs, device=dev, load=HostLoad(load, n, dev))
    op.coeffs, op.load = coeffs, load
    return fom_from_operator(op, int(z["probe"])), [float(f) for f in grid], op
