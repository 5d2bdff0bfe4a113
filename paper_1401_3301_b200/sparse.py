"""CSR output type, mirroring the reference ``SparseMatrix`` (sparse.py:42-73).

Canonical form: per row strictly increasing column indices, no stored
exact 0.0 (sparse.py:46-48); row_ptr/col_idx int64, vals f64.  When the
reference package is importable its class is used, so our drivers return
exactly the type the reference's own callers expect.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

try:  # pragma: no cover - depends on the environment
    from simplex_asm.sparse import SparseMatrix  # type: ignore
except Exception:

    @dataclass(frozen=True, eq=False)
    class SparseMatrix:  # type: ignore[no-redef]
        """Compressed sparse row matrix in canonical form."""

        nrows: int
        ncols: int
        row_ptr: np.ndarray  # (nrows+1,) int64
        col_idx: np.ndarray  # (nnz,) int64
        vals: np.ndarray     # (nnz,) float64

        @property
        def nnz(self) -> int:
            return len(self.vals)

        @property
        def shape(self) -> tuple[int, int]:
            return (self.nrows, self.ncols)

        def row_indices(self) -> np.ndarray:
            return np.repeat(np.arange(self.nrows, dtype=np.int64), np.diff(self.row_ptr))

        def to_dense(self) -> np.ndarray:
            out = np.zeros((self.nrows, self.ncols))
            out[self.row_indices(), self.col_idx] = self.vals
            return out


def to_scipy(a: SparseMatrix):
    """Zero-copy hand-off to scipy.sparse.csr_matrix."""
    import scipy.sparse

    return scipy.sparse.csr_matrix((a.vals, a.col_idx, a.row_ptr), shape=(a.nrows, a.ncols))


MM_HEADER = "%%MatrixMarket matrix coordinate real general"


def write_matrixmarket(a: SparseMatrix, path, chunk: int = 1 << 20) -> None:
    """MatrixMarket coordinate file, byte for byte the reference writer's
    output (sparse.py:208-219: real general header, one-based indices, values
    as ``%.17g``), formatted in chunks of ``chunk`` entries instead of one
    Python f-string per entry."""
    rp = np.asarray(a.row_ptr, dtype=np.int64)
    ci = np.asarray(a.col_idx, dtype=np.int64)
    va = np.asarray(a.vals, dtype=np.float64)
    rows = np.repeat(np.arange(a.nrows, dtype=np.int64), np.diff(rp))
    with open(path, "w") as f:
        f.write(MM_HEADER + "\n")
        f.write(f"{a.nrows} {a.ncols} {len(va)}\n")
        for s in range(0, len(va), chunk):
            e = min(s + chunk, len(va))
            f.write("".join(f"{i} {j} {v:.17g}\n" for i, j, v in
                            zip((rows[s:e] + 1).tolist(), (ci[s:e] + 1).tolist(), va[s:e].tolist())))


def empty_matrix(nrows: int, ncols: int) -> SparseMatrix:
    return SparseMatrix(nrows, ncols, np.zeros(nrows + 1, dtype=np.int64),
                        np.empty(0, dtype=np.int64), np.empty(0, dtype=np.float64))
