"""Thin torch-facing wrappers of the C-ABI linear-algebra entry points
(vb_csr_spmm, vb_csr_axpy_dense, vb_zgemm, vb_column_norms, vb_scale_columns).
All tensors are CUDA, complex128 row-major (2-D views with a row stride)."""

from __future__ import annotations

import torch

from . import _lib
from .assembly import DeviceCSR

CDT = torch.complex128


def _ld(t: torch.Tensor) -> int:
    if t.dim() == 1:
        return 1
    if t.stride(1) != 1:
        raise ValueError("row-major tensor with unit column stride expected")
    return t.stride(0)


def _cols(t: torch.Tensor) -> int:
    return 1 if t.dim() == 1 else t.shape[1]


RG_MIN_COLS = 3  # k from here takes the row-group SpMM (below: the SpMV / sub-warp CSR kernels)
RG_MIN_REUSE = 2.0


class RowGroups:
    """Row-group form of a CSR pattern (vb_csr_row_groups): built once per
    pattern on the host from the CSR arrays, kept on the device."""

    def __init__(self, n: int, indptr: torch.Tensor, indices: torch.Tensor):
        import ctypes
        import numpy as np
        lib = _lib.load()
        ip = np.ascontiguousarray(indptr.cpu().numpy(), dtype=np.int32)
        ix = np.ascontiguousarray(indices.cpu().numpy(), dtype=np.int32)
        nnz = max(int(ix.size), 1)
        lead = np.empty(max(n, 1), np.int32)
        rows = np.empty((max(n, 1), 8), np.int32)
        uoff = np.empty(max(n, 1), np.int32)
        masks = np.empty(nnz, np.uint8)
        vmap = np.empty((nnz, 8), np.int32)
        G, U = ctypes.c_int(0), ctypes.c_int64(0)
        hp = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
        _lib.check(lib.vb_csr_row_groups(n, hp(ip), hp(ix), hp(lead), hp(rows), hp(uoff), hp(masks), hp(vmap),
                                         ctypes.byref(G), ctypes.byref(U)), "vb_csr_row_groups")
        dev = indptr.device
        self.n_groups, self.n_union = G.value, U.value
        g, u = self.n_groups, self.n_union
        # X-row reuse of the grouping (nonzeros per gathered X row); below
        # RG_MIN_REUSE the dense 8-row blocks are mostly padding (e.g. a
        # row-restricted boundary matrix whose column ids are not its row ids)
        # and spmm keeps the CSR kernels
        self.reuse = int(ix.size) / max(u, 1)
        self.leader = torch.from_numpy(lead[:g].copy()).to(dev)
        self.rows = torch.from_numpy(rows[:g].copy()).to(dev)
        self.uoff = torch.from_numpy(uoff[:g].copy()).to(dev)
        self.masks = torch.from_numpy(masks[:u].copy()).to(dev)
        self.vmap = torch.from_numpy(vmap[:u].copy()).to(dev)

    def values(self, data: torch.Tensor) -> torch.Tensor:
        lib = _lib.load()
        gv = torch.empty((self.n_union, 8), dtype=torch.float64, device=data.device)
        _lib.check(lib.vb_rg_gather_values(self.n_union, _lib.ptr(self.vmap), _lib.ptr(data), _lib.ptr(gv),
                                           _lib.stream_handle()), "vb_rg_gather_values")
        return gv


def row_groups(A: DeviceCSR) -> RowGroups:
    """The pattern's row groups, cached on the pattern's indptr tensor (all
    primitives sharing a pattern share them)."""
    rg = getattr(A.indptr, "_vb_row_groups", None)
    if rg is None or rg[0] is not A.indices:
        rg = (A.indices, RowGroups(A.n, A.indptr, A.indices))
        A.indptr._vb_row_groups = rg
    return rg[1]


def _rg_values(A: DeviceCSR, rg: RowGroups) -> torch.Tensor:
    key = (A.data.data_ptr(), A.data._version, id(rg))
    c = getattr(A.data, "_vb_rg_vals", None)
    if c is None or c[0] != key:
        c = (key, rg.values(A.data))
        A.data._vb_rg_vals = c
    return c[1]


def spmm(A: DeviceCSR, X: torch.Tensor, alpha=1.0, beta=0.0, Y: torch.Tensor | None = None,
         path: str = "auto"):
    """Y = alpha A X + beta Y (A real CSR, X/Y complex).  Uniform-box primitives
    (A.kron set) with k >= 2 columns take the matrix-free Kronecker apply
    (vb_kron3_apply; same operator to rounding); other matrices with
    k >= RG_MIN_COLS columns the row-group SpMM (vb_rg_spmm, dense 8-row blocks on
    the FP64 tensor cores; equal to the CSR kernels to rounding), everything else the CSR SpMM (vb_csr_spmm).
    path: "auto", or "csr" / "rg" to force a CSR-form kernel."""
    lib = _lib.load()
    k = _cols(X)
    if Y is None:
        Y = torch.empty((A.n, k) if X.dim() == 2 else (A.n,), dtype=CDT, device=X.device)
        beta = 0.0
    ldx = _ld(X) if X.dim() == 2 else 1
    ldy = _ld(Y) if Y.dim() == 2 else 1
    kb = getattr(A, "kron", None)
    if path == "auto" and kb is not None and k >= 2:  # uniform-box primitive: matrix-free Kronecker apply
        _lib.check(lib.vb_kron3_apply(kb.npx, kb.npy, kb.npz, _lib.ptr(kb.K1), _lib.ptr(kb.M1), kb.maxnp,
                                      kb.stiff, k, _lib.zc(alpha), C_ptr(X), ldx, _lib.zc(beta), C_ptr(Y), ldy,
                                      _lib.stream_handle()), "vb_kron3_apply")
        return Y
    rg = row_groups(A) if path == "rg" or (path == "auto" and k >= RG_MIN_COLS) else None
    if rg is not None and (path == "rg" or rg.reuse >= RG_MIN_REUSE):
        gv = _rg_values(A, rg)
        _lib.check(lib.vb_rg_spmm(rg.n_groups, _lib.ptr(rg.leader), _lib.ptr(rg.rows), _lib.ptr(rg.uoff),
                                  _lib.ptr(A.indptr), _lib.ptr(A.indices), _lib.ptr(rg.masks), _lib.ptr(gv), k,
                                  C_ptr(X), ldx, C_ptr(Y), ldy, _lib.zc(alpha), _lib.zc(beta),
                                  _lib.stream_handle()), "vb_rg_spmm")
        return Y
    _lib.check(lib.vb_csr_spmm(A.n, _lib.ptr(A.indptr), _lib.ptr(A.indices), _lib.ptr(A.data), k,
                               C_ptr(X), ldx, C_ptr(Y), ldy, _lib.zc(alpha), _lib.zc(beta),
                               _lib.stream_handle()), "vb_csr_spmm")
    return Y


def C_ptr(t: torch.Tensor):
    import ctypes
    if not t.is_cuda:
        raise RuntimeError("vibro_b200: expected a CUDA tensor")
    return ctypes.c_void_p(t.data_ptr())


def axpy_dense(A: DeviceCSR, alpha, D: torch.Tensor):
    lib = _lib.load()
    _lib.check(lib.vb_csr_axpy_dense(A.n, _lib.ptr(A.indptr), _lib.ptr(A.indices), _lib.ptr(A.data),
                                     _lib.zc(alpha), C_ptr(D), _ld(D), _lib.stream_handle()),
               "vb_csr_axpy_dense")
    return D


def zgemm(transa: str, A: torch.Tensor, B: torch.Tensor, alpha=1.0, beta=0.0,
          C: torch.Tensor | None = None, m: int | None = None, n: int | None = None,
          k: int | None = None) -> torch.Tensor:
    """transa 'N': C = alpha A B + beta C;  'C': C = alpha A^H B + beta C."""
    lib = _lib.load()
    A2 = A if A.dim() == 2 else A.view(-1, 1)
    B2 = B if B.dim() == 2 else B.view(-1, 1)
    if transa == "N":
        m = A2.shape[0] if m is None else m
        k = A2.shape[1] if k is None else k
    else:
        k = A2.shape[0] if k is None else k
        m = A2.shape[1] if m is None else m
    n = B2.shape[1] if n is None else n
    if C is None:
        C = torch.empty((m, n), dtype=CDT, device=A.device)
        beta = 0.0
    C2 = C if C.dim() == 2 else C.view(-1, 1)
    ta = transa.encode()
    wb = lib.vb_zgemm_workspace_bytes(ta, m, n, k) if transa != "N" else 0  # 'N' takes no workspace
    # the workspace tensor must outlive the launch (another host thread could
    # otherwise be handed the freed block by the caching allocator)
    work = torch.empty(wb, dtype=torch.uint8, device=A.device) if wb else None
    _lib.check(lib.vb_zgemm(ta, m, n, k, _lib.zc(alpha), C_ptr(A2), _ld(A2), C_ptr(B2),
                            _ld(B2), _lib.zc(beta), C_ptr(C2), _ld(C2), C_ptr(work) if wb else None, wb,
                            _lib.stream_handle()), "vb_zgemm")
    del work
    return C


def zgemv_batched(items) -> None:
    """Y = alpha A X + beta Y for a list of (A, X, Y, alpha, beta) with X, Y
    (n, s) / (m, s) 2-D views, s <= 16 (vb_zgemv_batched: one launch per 32)."""
    if not items:
        return
    lib = _lib.load()
    arr = (_lib.VbGemvItem * len(items))()
    for i, (A, X, Y, alpha, beta) in enumerate(items):
        X2 = X if X.dim() == 2 else X.view(-1, 1)
        Y2 = Y if Y.dim() == 2 else Y.view(-1, 1)
        if A.shape[1] != X2.shape[0] or A.shape[0] != Y2.shape[0] or X2.shape[1] != Y2.shape[1]:
            raise ValueError("zgemv_batched: shape mismatch")
        arr[i] = _lib.VbGemvItem(A.shape[0], A.shape[1], X2.shape[1], 0, A.data_ptr(), _ld(A), X2.data_ptr(),
                                 _ld(X2), Y2.data_ptr(), _ld(Y2), _lib.zc(alpha), _lib.zc(beta))
    import ctypes
    _lib.check(lib.vb_zgemv_batched(len(items), ctypes.cast(arr, ctypes.c_void_p), _lib.stream_handle()),
               "vb_zgemv_batched")


def column_norms(W: torch.Tensor, m: int | None = None) -> torch.Tensor:
    lib = _lib.load()
    W2 = W if W.dim() == 2 else W.view(-1, 1)
    n = W2.shape[0]
    m = W2.shape[1] if m is None else m
    out = torch.empty(m, dtype=torch.float64, device=W.device)
    wb = lib.vb_column_norms_workspace_bytes(n, m)
    work = torch.empty(max(wb, 1), dtype=torch.uint8, device=W.device)
    _lib.check(lib.vb_column_norms(n, m, C_ptr(W2), _ld(W2), C_ptr(out), C_ptr(work), wb,
                                   _lib.stream_handle()), "vb_column_norms")
    return out


def scale_columns(W: torch.Tensor, scale: torch.Tensor, m: int | None = None):
    lib = _lib.load()
    W2 = W if W.dim() == 2 else W.view(-1, 1)
    m = W2.shape[1] if m is None else m
    sc = scale.to(torch.float64).contiguous()  # alive through the launch
    _lib.check(lib.vb_scale_columns(W2.shape[0], m, C_ptr(W2), _ld(W2), C_ptr(sc), _lib.stream_handle()),
               "vb_scale_columns")
    return W


BLOCK_GS_MAX = 16


def block_gs(W: torch.Tensor, Q: torch.Tensor, refs: torch.Tensor | None = None, tol: float = 0.0,
             reorth: float = 0.0, no_drop: bool = False, sync: bool = True):
    """Fused in-block Gram-Schmidt (vb_block_gs): the columns of W (n x kb,
    kb <= 16) orthogonalised twice against the kept ones and kept by the
    reference drop rule into Q[:, :nk].  Returns (nk, kept flags) — one host
    read per block."""
    lib = _lib.load()
    n, kb = W.shape
    kept = torch.empty(max(kb, 1), dtype=torch.int32, device=W.device)
    nk = torch.zeros(1, dtype=torch.int32, device=W.device)
    wb = lib.vb_block_gs_workspace_bytes()
    work = torch.empty(max(wb, 1), dtype=torch.uint8, device=W.device)
    refs_c = refs.contiguous() if refs is not None else None  # alive through the launch
    rp = _lib.ptr(refs_c) if refs_c is not None else None
    _lib.check(lib.vb_block_gs(n, kb, C_ptr(W), _ld(W), rp, tol, reorth, int(no_drop), C_ptr(Q), _ld(Q),
                               _lib.ptr(kept), _lib.ptr(nk), C_ptr(work), wb, _lib.stream_handle()),
               "vb_block_gs")
    if not sync:  # device tensors: the caller reads the counts later (one host sync for many blocks)
        return nk, kept[:kb]
    return int(nk.item()), kept[:kb].cpu().numpy()
