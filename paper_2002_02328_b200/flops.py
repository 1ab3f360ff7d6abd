"""Algorithmic work of the hot path, numpy/torch-free.

Kept free of torch and of the native library so bench.py's reference arm can
cost the reference's block step without mapping the product's .so.  The
operator module re-exports these (``blur.flops_*``).

* F_H = 2 * nnz(H rows): in-bounds taps only (zero-padded taps do not count);
  x/y factorise as n*k - r(r+1) per axis, z counts the taps inside [0, nz).
* The block-Jacobi sweep (bd3mg_jacobi_sweep) runs H over the residual rows,
  H^T over the block rows and the forward-only Gram (two block-embedded H per
  block, one with the hd-cache); the reference's own block step
  (objective.py:170-172 + 2x :258-260) runs H + H^T for the gradient and H +
  H^T per majorant product.
"""

from __future__ import annotations


def _axis(n: int, k: int) -> int:
    r = (k - 1) // 2
    return n * k - r * (r + 1)


def flops_H(dims, kdims, out_lo: int = 0, out_hi: int | None = None) -> int:
    """2*nnz of H rows [out_lo, out_hi] (dims = (nx, ny, nz), kdims = (kx, ky, kz))."""
    nx, ny, nz = dims
    kx, ky, kz = kdims
    if out_hi is None:
        out_hi = nz - 1
    rz = (kz - 1) // 2
    zt = sum(min(nz - 1, z + rz) - max(0, z - rz) + 1 for z in range(out_lo, out_hi + 1))
    return 2 * _axis(nx, kx) * _axis(ny, ky) * zt


def flops_H_embedded(dims, kdims, lo: int, hi: int) -> int:
    """H of a vector embedded on block rows [lo, hi] (zero elsewhere), over
    its nonzero output rows [lo-rz, hi+rz]: 2 * in-bounds taps whose input
    plane lies in the block."""
    nx, ny, nz = dims
    kx, ky, kz = kdims
    rz = (kz - 1) // 2
    zt = 0
    for zo in range(max(0, lo - rz), min(nz - 1, hi + rz) + 1):
        zt += min(hi, zo + rz) - max(lo, zo - rz) + 1
    return 2 * _axis(nx, kx) * _axis(ny, ky) * zt


def flops_jacobi_sweep(dims, kdims, blocks, hd_cache: bool = False, incremental: bool = False) -> int:
    """Correlation flops of one fused block-Jacobi sweep over ``blocks``
    (objects with z_lo / z_hi).  "hd-incremental" runs no residual
    correlation outside its refresh sweeps."""
    nz = dims[2]
    rz = (kdims[2] - 1) // 2
    lo = max(0, min(b.z_lo for b in blocks) - rz)
    hi = min(nz - 1, max(b.z_hi for b in blocks) + rz)
    f = 0 if incremental else flops_H(dims, kdims, lo, hi)
    hd_cache = hd_cache or incremental
    f += sum(flops_H(dims, kdims, b.z_lo, b.z_hi) for b in blocks)  # H^T rows: same tap count by symmetry
    gram = sum(flops_H_embedded(dims, kdims, b.z_lo, b.z_hi) for b in blocks)
    return f + (1 if hd_cache else 2) * gram


def ref_block_flops(dims, kdims, block_height: int) -> int:
    """Correlation flops of one reference block step on an interior block
    (reference arithmetic, objective.py:170-172 + 2x :258-260): H over the
    residual rows, H^T over the block, and two majorant products (H of the
    block-embedded vector, H^T back)."""
    nz = dims[2]
    rz = (kdims[2] - 1) // 2
    lo = (nz // 2 // block_height) * block_height
    hi = min(lo + block_height - 1, nz - 1)
    emb = flops_H_embedded(dims, kdims, lo, hi)
    return (flops_H(dims, kdims, max(0, lo - rz), min(nz - 1, hi + rz)) + flops_H(dims, kdims, lo, hi)
            + 2 * 2 * emb)
