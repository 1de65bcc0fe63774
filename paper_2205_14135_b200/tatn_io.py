"""Matrix test-vector IO in the reference's two interchangeable formats.

Restates ``proj/core/include/tatn/matrix_io.hpp:10-26`` / ``src/matrix_io.cpp``:

* CSV: one row per line, ',' separated, '.' decimal point, 17 significant digits
  (``std::to_chars(general, 17)`` == printf ``%.17g``), so binary64 round-trips exactly
  (matrix_io.cpp:53-60, 71-80). Reading trims blanks and a trailing CR, skips empty
  lines, rejects ragged rows and empty input (matrix_io.cpp:82-113).
* Binary: magic ``"TATN"``, u32 LE rows, u32 LE cols, rows*cols IEEE-754 binary64 LE,
  row-major (matrix_io.cpp:116-136). Bad magic / truncation raise like the reference's
  ``std::runtime_error``.

Used by the CLI (``paper_2205_14135_b200.cli``) to exchange golden vectors between the
CPU oracle and GPU runs; tests pin the bytes against the reference's own writer.
"""
from __future__ import annotations

import struct
from pathlib import Path

import numpy as np

MAGIC = b"TATN"


class MatrixIOError(RuntimeError):
    """The reference throws std::runtime_error for every IO failure (matrix_io.cpp)."""


def _as_matrix(m) -> np.ndarray:
    a = np.asarray(m, dtype=np.float64)
    if a.ndim != 2:
        raise MatrixIOError(f"matrix write: expected a 2-D matrix, got shape {a.shape}")
    return np.ascontiguousarray(a)


def to_binary_bytes(m) -> bytes:
    a = _as_matrix(m)
    return MAGIC + struct.pack("<II", a.shape[0], a.shape[1]) + a.astype("<f8").tobytes()


def from_binary_bytes(buf: bytes) -> np.ndarray:
    if len(buf) < 4 or buf[:4] != MAGIC:
        raise MatrixIOError("matrix read: bad magic (expected TATN)")
    if len(buf) < 12:
        raise MatrixIOError("matrix read: truncated header")
    rows, cols = struct.unpack_from("<II", buf, 4)
    n = rows * cols
    if len(buf) < 12 + 8 * n:
        raise MatrixIOError("matrix read: truncated payload")
    return np.frombuffer(buf, dtype="<f8", count=n, offset=12).astype(np.float64).reshape(rows, cols)


def write_matrix_binary(m, path) -> None:
    try:
        Path(path).write_bytes(to_binary_bytes(m))
    except OSError as e:
        raise MatrixIOError(f"cannot open for writing: {path}") from e


def read_matrix_binary(path) -> np.ndarray:
    try:
        buf = Path(path).read_bytes()
    except OSError as e:
        raise MatrixIOError(f"cannot open for reading: {path}") from e
    return from_binary_bytes(buf)


def to_csv_text(m) -> str:
    a = _as_matrix(m)
    return "".join(",".join(format(float(v), ".17g") for v in row) + "\n" for row in a)


def from_csv_text(text: str) -> np.ndarray:
    values, cols, rows = [], 0, 0
    for line in text.split("\n"):
        if line == "" or line == "\r":
            continue
        toks = [t.strip(" \t\r") for t in line.split(",")]
        try:
            row = [float(t) for t in toks]
        except ValueError as e:
            raise MatrixIOError(f"matrix read: bad CSV number in '{line}'") from e
        if rows == 0:
            cols = len(row)
        elif len(row) != cols:
            raise MatrixIOError("matrix read: ragged CSV rows")
        values.extend(row)
        rows += 1
    if rows == 0:
        raise MatrixIOError("matrix read: empty CSV")
    return np.asarray(values, dtype=np.float64).reshape(rows, cols)


def write_matrix_csv(m, path) -> None:
    try:
        Path(path).write_text(to_csv_text(m))
    except OSError as e:
        raise MatrixIOError(f"cannot open for writing: {path}") from e


def read_matrix_csv(path) -> np.ndarray:
    try:
        text = Path(path).read_text()
    except OSError as e:
        raise MatrixIOError(f"cannot open for reading: {path}") from e
    return from_csv_text(text)
