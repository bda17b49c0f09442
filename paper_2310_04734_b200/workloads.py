"""Seeded synthetic inputs with the shapes of BASELINE.json's configs (host-side
input generation; no datasets exist for this path).

cfg5 "reduced-sweep throughput stress": dense complex128 reduced matrices
  K_r = sigma_K (X X^H / r + I) (1 + i eta)     Hermitian PD plus i eta K
  M_r = Y Y^H / r + I                            Hermitian PD
  D_r = sigma_D U U^H / r,   U: r x 32           low rank 32
  B   : r x 16 RHS, entries N(0,1) + i N(0,1)
  C_R : 50 x r output rows, entries N(0,1) + i N(0,1)
  f   = linspace(1, 1000, 100000)
The construction mirrors tests/test_mor.py:26-37 (frozen_fom); sigma_K places
the undamped eigenfrequencies (~134–670 Hz) inside the swept band so the LU
pivots through resonances, and sigma_D is a 5 %-of-critical viscous scale.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

CFG5_ORDERS = (256, 1024, 2048)
CFG5_NFREQ = 100_000
CFG5_RHS = 16
CFG5_NOUT = 50
CFG5_DRANK = 32
CFG5_ETA = 0.02


@dataclass
class ReducedWorkload:
    name: str
    prims: np.ndarray      # (3, r, r): [K_r (1+i eta), D_r, M_r]
    kinds: tuple           # ('K', 'D', 'M') — alpha = [1, i w, -w^2]
    b: np.ndarray          # (r, s)
    c_r: np.ndarray        # (n_out, r)
    freqs: np.ndarray      # (F,)
    seed: int

    @property
    def r(self):
        return self.prims.shape[1]

    def alpha(self, freqs=None) -> np.ndarray:
        f = self.freqs if freqs is None else np.asarray(freqs, float)
        w = 2.0 * math.pi * f
        cols = {"K": np.ones_like(w, dtype=complex), "D": 1j * w, "M": -(w * w) + 0j}
        return np.stack([cols[k] for k in self.kinds], axis=1)


def _cn(rng, *shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def cfg5(r: int = 1024, n_freq: int = CFG5_NFREQ, s: int = CFG5_RHS, n_out: int = CFG5_NOUT,
         seed: int = 5, f_lo: float = 1.0, f_hi: float = 1000.0) -> ReducedWorkload:
    rng = np.random.default_rng(seed)
    sig_k = (2.0 * math.pi * 300.0) ** 2
    X = _cn(rng, r, r)
    Y = _cn(rng, r, r)
    M = Y @ Y.conj().T / r + np.eye(r)
    U = _cn(rng, r, CFG5_DRANK)
    sig_d = 2 * 0.05 * (2.0 * math.pi * 300.0)
    D = sig_d * (U @ U.conj().T) / r
    # enforce exact Hermitian symmetry of the PD parts (rounding of X X^H)
    M = 0.5 * (M + M.conj().T)
    D = 0.5 * (D + D.conj().T)
    Kh = sig_k * (X @ X.conj().T / r + np.eye(r))
    K = 0.5 * (Kh + Kh.conj().T) * (1 + 1j * CFG5_ETA)
    B = _cn(rng, r, s)
    C = _cn(rng, n_out, r)
    freqs = np.linspace(f_lo, f_hi, n_freq)
    return ReducedWorkload(name=f"cfg5_r{r}", prims=np.stack([K, D, M]), kinds=("K", "D", "M"),
                           b=B, c_r=C, freqs=freqs, seed=seed)


def _without(sorted_ids: np.ndarray, drop) -> np.ndarray:
    """np.setdiff1d(sorted_ids, drop) for a sorted unique id array, without the
    O(n log n) re-sort (376k interior nodes at cfg3)."""
    keep = np.ones(len(sorted_ids), dtype=bool)
    pos = np.searchsorted(sorted_ids, np.asarray(drop))
    pos = pos[(pos < len(sorted_ids))]
    keep[pos[sorted_ids[pos] == np.asarray(drop)[: len(pos)]]] = False
    return sorted_ids[keep]


def cfg5_eigenfrequencies(w: ReducedWorkload) -> np.ndarray:
    """Undamped eigenfrequencies (Hz) of a cfg5 workload: K_h x = w^2 M x with
    K_h = K_r / (1 + i eta) Hermitian PD (host, scipy eigh).  The frequencies
    next to these are where the reduced LU pivots hardest (parity probes)."""
    import scipy.linalg as sla
    Kh = w.prims[0] / (1 + 1j * CFG5_ETA)
    Kh = 0.5 * (Kh + Kh.conj().T)
    M = w.prims[2]
    lam = sla.eigh(Kh, 0.5 * (M + M.conj().T), eigvals_only=True)
    return np.sqrt(np.maximum(lam, 0.0)) / (2.0 * math.pi)


# ---------------------------------------------------------------- cfg1 -----
CFG1_BOX = (0.0, 0.0, 0.0, 2.0, 1.6, 1.2)
CFG1_NE = (10, 8, 6)
AIR_RHO, AIR_C = 1.21, 343.0
CFG1_Z = AIR_RHO * AIR_C * (5 + 1j)
CFG1_POINTS = (42.5, 87.5, 132.5, 177.5)   # quartile midpoints of [20, 200]
CFG1_MOMENTS = 8
CFG1_NREC = 50


def cfg1_layout(seed: int = 1, box=CFG1_BOX, ne=CFG1_NE, n_rec: int = CFG1_NREC):
    """Host-side layout of cfg1: mesh, seeded source node and receivers.

    Source: one seeded interior node; receivers: n_rec distinct seeded interior
    nodes excluding the source."""
    from .assembly import hex27_box, interior_nodes
    xyz, conn = hex27_box(box, *ne)
    inner = interior_nodes(xyz, box)
    rng = np.random.default_rng(seed)
    src = int(rng.choice(inner))
    rec = np.sort(rng.choice(_without(inner, [src]), n_rec, replace=False)).astype(np.int64)
    return xyz, conn, src, rec


def cfg1_model(seed: int = 1, box=CFG1_BOX, ne=CFG1_NE, n_rec: int = CFG1_NREC, device=None,
               fdm: bool = False):
    """cfg1 (BASELINE configs[0]): rigid air box 2.0 x 1.6 x 1.2 m, 10 x 8 x 6
    hex27 Helmholtz elements (n = 4641), floor impedance Z = rho c (5 + 1i),
    unit point source, 50 receivers.  All primitives assembled on the GPU;
    returns (FullOrderModel with an affine operator, layout dict).  Full-order
    solves use the dense GPU LU (the reference's direct solve, mor.py:48-49)
    or, with `fdm`, the box fast-diagonalisation solver (one impedance wall:
    exact Kronecker sum) refined to the same 1e-10 residual contract."""
    import torch
    from . import assembly
    from .mor import AffineOperator, AffineTerm, FullOrderModel
    xyz, conn, src, rec = cfg1_layout(seed, box, ne, n_rec)
    Kg, Mn = assembly.assemble_helmholtz(xyz, conn, device)
    F = assembly.assemble_face_mass(xyz, assembly.hex27_box_face(ne, "z0", conn), device)
    n = xyz.shape[0]
    b = torch.zeros(n, dtype=torch.complex128, device=Kg.data.device)
    b[src] = 1.0
    C = np.zeros((len(rec), n))
    C[np.arange(len(rec)), rec] = 1.0
    aff = AffineOperator(K=[AffineTerm(Kg, 1.0 / AIR_RHO)],
                         M=[AffineTerm(Mn, 1.0 / (AIR_RHO * AIR_C * AIR_C))],
                         D=[AffineTerm(F, 1.0 / CFG1_Z)], load=b)
    fdm_solver = None
    if fdm:
        from .fdm import BoxFDM
        fdm_solver = BoxFDM(box, ne, AIR_RHO, AIR_C, {"z0": CFG1_Z})
    fom = FullOrderModel(c_out=C, n=n, affine=aff, fdm=fdm_solver, prefer_fdm=fdm)
    return fom, {"xyz": xyz, "conn": conn, "src": src, "rec": rec, "Kg": Kg, "Mn": Mn, "F": F,
                 "freqs": np.arange(20.0, 200.5, 1.0), "points": CFG1_POINTS,
                 "moments": CFG1_MOMENTS}


# ---------------------------------------------------------------- cfg3 -----
CFG3_BOX = (0.0, 0.0, 0.0, 6.0, 3.0, 2.5)
CFG3_NE = (60, 30, 25)
CFG3_WALLS = ("x0", "y1", "z1")                 # three absorbing walls (recorded choice)
# 10 points x 5 moments x 8 sources -> r = 400 (BASELINE), points denser toward
# the top of the band where the modal density grows (~f^2): certified on a
# disjoint grid at eps_max 1.3e-3 pointwise over all 50 x 8 outputs (reference
# tol 1e-2, tests/test_acceptance.py:272-305).  The 5 x 10 quintile-midpoint
# choice of round 1 reached only 5.0 pointwise / 3.7e-2 normwise at 300 Hz.
CFG3_POINTS = (30.0, 70.0, 110.0, 150.0, 185.0, 215.0, 240.0, 262.0, 282.0, 298.0)
CFG3_MOMENTS = 5
CFG3_NSRC = 8


def cfg3_model(seed: int = 3, box=CFG3_BOX, ne=CFG3_NE, n_src: int = CFG3_NSRC, n_rec: int = CFG1_NREC,
               device=None, per_element_z: bool = False):
    """cfg3 (BASELINE configs[2]): 6 x 3 x 2.5 m air box, 60 x 30 x 25 hex27
    (n = 376,431, nnz = 23,300,121), three absorbing walls with seeded
    Z_w = rho c U[2, 10] (real, one value per wall — keeps the FDM solver
    exact), 8 seeded interior point sources (block RHS), 50 receivers,
    20:0.25:300 Hz.  Returns (FullOrderModel with affine operator + BoxFDM, layout)."""
    import torch
    from . import assembly
    from .fdm import BoxFDM
    from .mor import AffineOperator, AffineTerm, FullOrderModel
    rng = np.random.default_rng(seed)
    xyz, conn = assembly.hex27_box(box, *ne)
    inner = assembly.interior_nodes(xyz, box)
    src = np.sort(rng.choice(inner, n_src, replace=False)).astype(np.int64)
    rec = np.sort(rng.choice(_without(inner, src), n_rec, replace=False)).astype(np.int64)
    Zs = {w: AIR_RHO * AIR_C * float(rng.uniform(2.0, 10.0)) for w in CFG3_WALLS}
    # structured box: the vb_hex27_box_csr CSR (same pattern as the general
    # assembly, values to rounding) carrying the Kronecker form, so the
    # projections P V run matrix-free (vb_kron3_apply)
    Kg, Mn = assembly.assemble_helmholtz_box(box, ne, device)
    n = xyz.shape[0]
    D_terms = []
    iterative, Ze = None, {}
    if per_element_z:
        # seeded Z_e = rho c U[2, 10] per wall face element (separate stream, so
        # sources / receivers stay those of the per-wall model); the walls enter
        # as D_w = sum_e F_e / Z_e and the full-order solver becomes GMRES
        # preconditioned by the box FDM with per-wall harmonic-mean impedances
        from .fdm import BoxFDM
        from .gmres import BoxGmres
        rz = np.random.default_rng(seed + 1000)
        zmean = {}
        for w in CFG3_WALLS:
            fc = assembly.hex27_box_face(ne, w, conn)
            Ze[w] = AIR_RHO * AIR_C * rz.uniform(2.0, 10.0, len(fc))
            D_terms.append(AffineTerm(assembly.assemble_weighted_face_mass(xyz, fc, 1.0 / Ze[w], device), 1.0))
            zmean[w] = 1.0 / float(np.mean(1.0 / Ze[w]))
        iterative = BoxGmres(BoxFDM(box, ne, AIR_RHO, AIR_C, zmean))
    else:
        for w, Z in Zs.items():
            F = assembly.assemble_face_mass(xyz, assembly.hex27_box_face(ne, w, conn), device)
            D_terms.append(AffineTerm(F, 1.0 / Z))
    b = torch.zeros((n, n_src), dtype=torch.complex128, device=Kg.data.device)
    b[torch.as_tensor(src, device=b.device), torch.arange(n_src, device=b.device)] = 1.0
    C = np.zeros((n_rec, n))
    C[np.arange(n_rec), rec] = 1.0
    aff = AffineOperator(K=[AffineTerm(Kg, 1.0 / AIR_RHO)],
                         M=[AffineTerm(Mn, 1.0 / (AIR_RHO * AIR_C * AIR_C))], D=D_terms, load=b)
    fom = FullOrderModel(c_out=C, n=n, affine=aff, fdm=None if per_element_z else BoxFDM(box, ne, AIR_RHO, AIR_C, Zs),
                         iterative=iterative)
    return fom, {"xyz": xyz, "conn": conn, "src": src, "rec": rec, "walls": Zs, "Kg": Kg, "Mn": Mn, "Z_e": Ze,
                 "freqs": np.arange(20.0, 300.0 + 1e-9, 0.25), "points": CFG3_POINTS,
                 "moments": CFG3_MOMENTS}


# ---------------------------------------------------------------- cfg2 -----
CFG2_PLATE = dict(E=60e9, nu=0.3, rho=1550.0, t=0.003)
CFG2_BOX = (0.0, 0.0, 0.0, 0.8, 0.6, 0.5)
CFG2_NE = (16, 12, 10)
CFG2_THETA = math.radians(30.0)
# r = 60 as BASELINE's 6 x 10, spread over 10 points x 6 moments: eps_max
# 3.8e-3 on a disjoint grid (6 sextile midpoints x 10 moments: 0.44 at 427 Hz)
CFG2_POINTS = (40.0, 100.0, 160.0, 220.0, 280.0, 330.0, 380.0, 420.0, 460.0, 495.0)
CFG2_MOMENTS = 6


def cfg2_model(seed: int = 2, box=CFG2_BOX, ne=CFG2_NE, n_rec: int = CFG1_NREC, device=None,
               use_schur: bool = True):
    """cfg2 (BASELINE configs[1]): clamped 0.8 x 0.6 m, 3 mm CFRP-like plate of
    16 x 12 9-node Reissner-Mindlin + membrane elements on top of a 0.8 x 0.6 x 0.5 m
    air cavity of 16 x 12 x 10 hex27 (conforming wet face), eta(f) = 0.01 + 2e-5 f
    on the plate stiffness, unit plane-wave pressure at 30 deg incidence, 50
    seeded cavity receivers, 20:0.5:500 Hz, r = 60 (10 points x 6 moments).
    DoFs: [plate free (u, v, w, bx, by) | cavity pressure]; n = 3,565 + 17,325."""
    import torch
    from . import assembly, plate
    from .mor import AffineOperator, AffineTerm, FullOrderModel
    dev = torch.device(device or "cuda")
    nx, ny, nz = ne
    x0, y0, z0, x1, y1, z1 = box
    xyz_f, conn_f = assembly.hex27_box(box, *ne)
    pxyz, pconn = plate.plate_mesh((x0, y0, x1, y1), nx, ny, z1)
    dmap, n_p = plate.clamped_dof_map(nx, ny)
    n_f = xyz_f.shape[0]
    n = n_p + n_f
    # cavity primitives in the global numbering (rows/cols offset by the plate DoFs)
    conn_g = (conn_f + n_p).astype(np.int32)
    xyz_d = torch.as_tensor(xyz_f, device=dev)
    Ke, Me = assembly.hex27_helmholtz(xyz_d, torch.as_tensor(conn_f, device=dev))
    Kg = plate.assemble_blocks(n, n, conn_g, conn_g, Ke, dev)
    Mn = plate.assemble_blocks(n, n, conn_g, conn_g, Me, dev)
    # plate
    P = CFG2_PLATE
    Kpe, Mpe = plate.plate_elements(torch.as_tensor(pxyz, device=dev), torch.as_tensor(pconn, device=dev),
                                    P["E"], P["nu"], P["rho"], P["t"])
    pd = dmap[pconn].reshape(len(pconn), 45)
    Kp = plate.assemble_blocks(n, n, pd, pd, Kpe, dev)
    Mp = plate.assemble_blocks(n, n, pd, pd, Mpe, dev)
    # coupling on the wet face (plate element e <-> cavity top-face element e)
    fconn = assembly.hex27_box_face(ne, "z1", conn_f)
    Fe = assembly.face_mass(torch.as_tensor(pxyz, device=dev), torch.as_tensor(pconn, device=dev))
    wd = dmap[pconn][:, :, 2]
    Fsf = plate.assemble_blocks(n, n, wd, fconn + n_p, Fe, dev)
    Ffs = plate.assemble_blocks(n, n, fconn + n_p, wd, Fe.transpose(1, 2).contiguous(), dev)
    sgn = -1.0  # structure -> fluid normal is -z (cavity below the plate)
    rng = np.random.default_rng(seed)
    inner = assembly.interior_nodes(xyz_f, box)
    rec = np.sort(rng.choice(inner, n_rec, replace=False)).astype(np.int64) + n_p
    Cmat = np.zeros((n_rec, n))
    Cmat[np.arange(n_rec), rec] = 1.0
    load = plate.PlaneWaveLoad(pxyz, pconn, dmap, n, AIR_C, CFG2_THETA, 1.0, dev)
    aff = AffineOperator(
        K=[AffineTerm(Kg, 1.0 / AIR_RHO), AffineTerm(Kp, lambda f: 1.0 + 1j * plate.eta_cfg2(f)),
           AffineTerm(Fsf, -sgn)],
        M=[AffineTerm(Mn, 1.0 / (AIR_RHO * AIR_C * AIR_C)), AffineTerm(Mp, 1.0), AffineTerm(Ffs, AIR_RHO * sgn)],
        D=[], load=load)
    # cavity block = box operator with rigid walls -> Schur complement on the plate
    from .fdm import BoxFDM
    from .schur import CoupledBoxSchur
    schur = CoupledBoxSchur(aff, n_p, BoxFDM(box, ne, AIR_RHO, AIR_C, {}), dev) if use_schur else None
    fom = FullOrderModel(c_out=Cmat, n=n, affine=aff, schur=schur)
    return fom, {"n_plate": n_p, "n_fluid": n_f, "rec": rec, "dmap": dmap, "pxyz": pxyz, "pconn": pconn,
                 "xyz_f": xyz_f, "conn_f": conn_f, "fconn": fconn, "Kg": Kg, "Mn": Mn, "Kp": Kp, "Mp": Mp,
                 "Fsf": Fsf, "Ffs": Ffs, "load": load, "freqs": np.arange(20.0, 500.0 + 1e-9, 0.5),
                 "points": CFG2_POINTS, "moments": CFG2_MOMENTS}
