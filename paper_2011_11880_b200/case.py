"""Columnar raw case: the network description ``build_system`` consumes.

Mirrors the reference's ``RawCase`` (pflow/case_io.py:24-68) field for field,
but stores each MATPOWER column as one numpy array instead of a list of row
records, so 200k-bus synthetic grids build in milliseconds.  The reference's
own ``RawCase`` objects are accepted through :func:`from_rows`;
``parse_case``/``parse_case_file``/``write_case`` read and write the MATPOWER
numeric subset directly.

``validate_case`` restates pflow/case_io.py:189-232 (same violation codes and
row indices) vectorised.
"""

from __future__ import annotations

import re
from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Violation:
    """One structural-invariant violation (pflow/case_io.py:71-77)."""

    code: str
    row: int
    message: str


@dataclass(frozen=True)
class RawCase:
    """Verbatim network tables (no unit conversion), one array per column.

    bus:    bus_id, bus_type (1 PQ, 2 PV, 3 slack), pd, qd (MW/MVAr), gs, bs,
            vm (pu), va (degrees), base_kv
    gen:    gen_bus (bus id), pg, qg, qmax, qmin, vg, gen_status
    branch: from_bus, to_bus (bus ids), r, x, b (pu), ratio (0 already
            mapped to 1.0 as in pflow/case_io.py:156), angle (degrees),
            br_status
    """

    base_mva: float
    bus_id: np.ndarray
    bus_type: np.ndarray
    pd: np.ndarray
    qd: np.ndarray
    gs: np.ndarray
    bs: np.ndarray
    vm: np.ndarray
    va: np.ndarray
    base_kv: np.ndarray
    gen_bus: np.ndarray
    pg: np.ndarray
    qg: np.ndarray
    qmax: np.ndarray
    qmin: np.ndarray
    vg: np.ndarray
    gen_status: np.ndarray
    from_bus: np.ndarray
    to_bus: np.ndarray
    r: np.ndarray
    x: np.ndarray
    b: np.ndarray
    ratio: np.ndarray
    angle: np.ndarray
    br_status: np.ndarray
    name: str = ""

    @property
    def n_bus(self) -> int:
        return int(self.bus_id.shape[0])

    @property
    def n_gen(self) -> int:
        return int(self.gen_bus.shape[0])

    @property
    def n_branch(self) -> int:
        return int(self.from_bus.shape[0])

    def to_arrays(self) -> dict:
        """Flat dict of the columns (for ``np.savez`` fixtures)."""
        out = {k: getattr(self, k) for k in _COLUMNS}
        out["base_mva"] = np.float64(self.base_mva)
        return out

    @staticmethod
    def from_arrays(d, name: str = "") -> "RawCase":
        kw = {k: np.asarray(d[k]) for k in _COLUMNS}
        return RawCase(base_mva=float(d["base_mva"]), name=name, **kw)


_COLUMNS = ("bus_id", "bus_type", "pd", "qd", "gs", "bs", "vm", "va", "base_kv",
            "gen_bus", "pg", "qg", "qmax", "qmin", "vg", "gen_status",
            "from_bus", "to_bus", "r", "x", "b", "ratio", "angle", "br_status")


def make_case(base_mva, bus, gen, branch, name: str = "") -> RawCase:
    """Build a RawCase from three column dicts (keys as in :class:`RawCase`)."""
    f8 = lambda a: np.ascontiguousarray(a, dtype=np.float64)
    i8 = lambda a: np.ascontiguousarray(a, dtype=np.int64)
    return RawCase(
        base_mva=float(base_mva),
        bus_id=i8(bus["bus_id"]), bus_type=i8(bus["bus_type"]),
        pd=f8(bus["pd"]), qd=f8(bus["qd"]), gs=f8(bus["gs"]), bs=f8(bus["bs"]),
        vm=f8(bus["vm"]), va=f8(bus["va"]), base_kv=f8(bus["base_kv"]),
        gen_bus=i8(gen["gen_bus"]), pg=f8(gen["pg"]), qg=f8(gen["qg"]),
        qmax=f8(gen["qmax"]), qmin=f8(gen["qmin"]), vg=f8(gen["vg"]),
        gen_status=i8(gen["gen_status"]),
        from_bus=i8(branch["from_bus"]), to_bus=i8(branch["to_bus"]),
        r=f8(branch["r"]), x=f8(branch["x"]), b=f8(branch["b"]),
        ratio=f8(branch["ratio"]), angle=f8(branch["angle"]),
        br_status=i8(branch["br_status"]),
        name=name,
    )


def from_rows(raw) -> RawCase:
    """Convert a reference ``pflow.RawCase`` (row records) to columns."""
    bus = {
        "bus_id": [r.bus_id for r in raw.bus_rows],
        "bus_type": [r.bus_type for r in raw.bus_rows],
        "pd": [r.pd for r in raw.bus_rows], "qd": [r.qd for r in raw.bus_rows],
        "gs": [r.gs for r in raw.bus_rows], "bs": [r.bs for r in raw.bus_rows],
        "vm": [r.vm for r in raw.bus_rows], "va": [r.va for r in raw.bus_rows],
        "base_kv": [r.base_kv for r in raw.bus_rows],
    }
    gen = {
        "gen_bus": [g.bus_id for g in raw.gen_rows], "pg": [g.pg for g in raw.gen_rows],
        "qg": [g.qg for g in raw.gen_rows], "qmax": [g.qmax for g in raw.gen_rows],
        "qmin": [g.qmin for g in raw.gen_rows], "vg": [g.vg for g in raw.gen_rows],
        "gen_status": [g.status for g in raw.gen_rows],
    }
    br = {
        "from_bus": [b.from_bus for b in raw.branch_rows],
        "to_bus": [b.to_bus for b in raw.branch_rows],
        "r": [b.r for b in raw.branch_rows], "x": [b.x for b in raw.branch_rows],
        "b": [b.b for b in raw.branch_rows], "ratio": [b.ratio for b in raw.branch_rows],
        "angle": [b.angle for b in raw.branch_rows],
        "br_status": [b.status for b in raw.branch_rows],
    }
    return make_case(raw.base_mva, bus, gen, br, name=getattr(raw, "name", ""))


def to_rows(case: RawCase):
    """Convert to the reference's row-record ``RawCase`` (needs ``pflow``)."""
    from pflow.case_io import BranchRow, BusRow, GenRow
    from pflow.case_io import RawCase as RefRawCase

    buses = [BusRow(int(case.bus_id[i]), int(case.bus_type[i]), float(case.pd[i]),
                    float(case.qd[i]), float(case.gs[i]), float(case.bs[i]),
                    float(case.vm[i]), float(case.va[i]), float(case.base_kv[i]))
             for i in range(case.n_bus)]
    gens = [GenRow(int(case.gen_bus[i]), float(case.pg[i]), float(case.qg[i]),
                   float(case.qmax[i]), float(case.qmin[i]), float(case.vg[i]),
                   int(case.gen_status[i]))
            for i in range(case.n_gen)]
    brs = [BranchRow(int(case.from_bus[i]), int(case.to_bus[i]), float(case.r[i]),
                     float(case.x[i]), float(case.b[i]), float(case.ratio[i]),
                     float(case.angle[i]), int(case.br_status[i]))
           for i in range(case.n_branch)]
    return RefRawCase(case.base_mva, buses, gens, brs, name=case.name)


def validate_case(raw: RawCase) -> list[Violation]:
    """Structural checks; same codes/rows as pflow/case_io.py:189-232."""
    out: list[Violation] = []
    if raw.base_mva <= 0:
        out.append(Violation("NONPOSITIVE_BASE_MVA", -1,
                             f"baseMVA must be positive, got {raw.base_mva}"))
    ids = raw.bus_id
    for i in np.flatnonzero(~np.isin(raw.bus_type, (1, 2, 3))):
        out.append(Violation("INVALID_BUS_TYPE", int(i),
                             f"bus {int(ids[i])} has unsupported type {int(raw.bus_type[i])}"))
    slack_rows = np.flatnonzero(raw.bus_type == 3)
    if slack_rows.size == 0:
        out.append(Violation("MISSING_SLACK", -1, "no type-3 (slack) bus"))
    for i in slack_rows[1:]:
        out.append(Violation("MULTIPLE_SLACK", int(i),
                             f"bus {int(ids[i])} is a second type-3 bus"))
    gen_known = np.isin(raw.gen_bus, ids)
    for i in np.flatnonzero(~gen_known):
        out.append(Violation("UNKNOWN_BUS", int(i),
                             f"gen {int(i)} references unknown bus {int(raw.gen_bus[i])}"))
    slack_ids = ids[slack_rows]
    slack_has_gen = bool(np.any(gen_known & np.isin(raw.gen_bus, slack_ids)
                                & (raw.gen_status != 0)))
    if slack_rows.size and not slack_has_gen:
        out.append(Violation("SLACK_WITHOUT_GEN", int(slack_rows[0]),
                             "slack bus has no in-service generator"))
    br_known = np.isin(raw.from_bus, ids) & np.isin(raw.to_bus, ids)
    zero_z = (raw.br_status != 0) & (raw.r * raw.r + raw.x * raw.x == 0.0)
    for i in range(raw.n_branch) if (~br_known | zero_z).any() else ():
        if not br_known[i]:
            out.append(Violation("UNKNOWN_BUS", i, f"branch {i} references unknown bus"))
        if zero_z[i]:
            out.append(Violation("ZERO_IMPEDANCE", i, f"in-service branch {i} has r = x = 0"))
    return out


# ---------------------------------------------------------------------------
# MATPOWER case text (on-disk input)
# ---------------------------------------------------------------------------

class CaseFormatError(ValueError):
    """Malformed case text; ``line`` is 1-based when known (pflow/case_io.py:16-21)."""

    def __init__(self, message: str, line: int = 0):
        super().__init__(f"line {line}: {message}" if line else message)
        self.line = line


# minimum columns consumed per MATPOWER v2 matrix
_MIN_COLS = {"bus": 10, "gen": 8, "branch": 11}

# one assignment statement: "<lhs> = <rhs>" (lhs up to the first '=')
_ASSIGNMENT = re.compile(r"^([^=]+?)\s*=\s*(.*?)\s*$")


def _code_lines(text: str):
    """(line number, code) of every line that holds code: '%' comments are
    dropped, surrounding blanks stripped, empty lines skipped."""
    for lineno, line in enumerate(text.splitlines(), start=1):
        code = line.partition("%")[0].strip()
        if code:
            yield lineno, code


class _Table:
    """Rows of one matrix as they arrive.  A row ends at ';', at the end of a
    line or at the closing ']'; text after ']' on that line is ignored."""

    def __init__(self, key: str):
        self.key = key
        self.rows: list[list[float]] = []
        self.lines: list[int] = []

    def take(self, lineno: int, code: str) -> bool:
        """Consume one line of the matrix body; True once it is closed."""
        body, bracket, _ = code.partition("]")
        for segment in body.split(";"):
            toks = segment.split()
            if toks:
                self.rows.append(self._numbers(toks, lineno))
                self.lines.append(lineno)
        return bool(bracket)

    def _numbers(self, toks: list[str], lineno: int) -> list[float]:
        need = _MIN_COLS[self.key]
        if len(toks) < need:
            raise CaseFormatError(f"matrix {self.key!r} row has {len(toks)} columns, "
                                  f"needs at least {need}", lineno)
        out = []
        for t in toks:
            try:
                out.append(float(t))
            except ValueError:
                raise CaseFormatError(f"non-numeric token {t!r} in matrix {self.key!r}",
                                      lineno) from None
        return out

    def column(self, j: int, dtype=np.float64) -> np.ndarray:
        return np.array([r[j] for r in self.rows], dtype=np.float64).astype(dtype)


def parse_case(text: str, name: str = "") -> RawCase:
    """Parse the numeric-matrix subset of MATPOWER v2 case text.

    Accepts ``baseMVA`` and the ``bus``/``gen``/``branch`` assignments
    (``mpc.`` prefix optional), ``%`` comments, rows ended by ``;`` or a
    newline.  Other assignments (``version``, ``gencost``, ...) are skipped.
    The error conditions and messages are pflow's (case_io.py:85-158, so a
    caller's error handling carries over): malformed matrix, non-numeric
    token, too few columns, missing baseMVA or matrix, matrix assigned twice,
    duplicate bus id - each with its line number.  A tap ratio of 0 becomes
    1.0 (MATPOWER convention).
    """
    base_mva = None
    tables: dict[str, _Table] = {}
    open_table: _Table | None = None
    for lineno, code in _code_lines(text):
        if open_table is not None:
            if open_table.take(lineno, code):
                open_table = None
            continue
        m = _ASSIGNMENT.match(code)
        if m is None:
            continue                       # function header, other statements
        key = m.group(1).rsplit(".", 1)[-1]
        value = m.group(2)
        if key == "baseMVA":
            number = value.rstrip(";").strip()
            try:
                base_mva = float(number)
            except ValueError:
                raise CaseFormatError(f"baseMVA is not numeric: {number!r}", lineno) from None
        elif key in _MIN_COLS:
            if not value.startswith("["):
                raise CaseFormatError(f"expected '[' to open matrix {key!r}", lineno)
            if key in tables:
                raise CaseFormatError(f"matrix {key!r} assigned twice", lineno)
            open_table = tables[key] = _Table(key)
            if open_table.take(lineno, value[1:]):
                open_table = None
    if open_table is not None:
        raise CaseFormatError(f"matrix {open_table.key!r} is never closed with '];'",
                              len(text.splitlines()))
    if base_mva is None:
        raise CaseFormatError("missing required scalar 'baseMVA'")
    for key in ("bus", "gen", "branch"):
        if key not in tables:
            raise CaseFormatError(f"missing required matrix '{key}'")
    bus, gen, br = tables["bus"], tables["gen"], tables["branch"]
    ids = bus.column(0, np.int64)
    uniq, first, counts = np.unique(ids, return_index=True, return_counts=True)
    if (counts > 1).any():   # report the first repeated row in file order
        seen_first = np.zeros(ids.size, bool)
        seen_first[first] = True
        dup = int(np.flatnonzero(~seen_first)[0])
        raise CaseFormatError(f"duplicate bus id {int(ids[dup])}", bus.lines[dup])
    ratio = br.column(8)
    return make_case(
        base_mva,
        {"bus_id": ids, "bus_type": bus.column(1, np.int64), "pd": bus.column(2),
         "qd": bus.column(3), "gs": bus.column(4), "bs": bus.column(5), "vm": bus.column(7),
         "va": bus.column(8), "base_kv": bus.column(9)},
        {"gen_bus": gen.column(0, np.int64), "pg": gen.column(1), "qg": gen.column(2),
         "qmax": gen.column(3), "qmin": gen.column(4), "vg": gen.column(5),
         "gen_status": gen.column(7, np.int64)},
        {"from_bus": br.column(0, np.int64), "to_bus": br.column(1, np.int64),
         "r": br.column(2), "x": br.column(3), "b": br.column(4),
         "ratio": np.where(ratio != 0.0, ratio, 1.0), "angle": br.column(9),
         "br_status": br.column(10, np.int64)},
        name=name)


def parse_case_file(path) -> RawCase:
    """Read and parse a MATPOWER case file (UTF-8); the case is named after the file."""
    from pathlib import Path

    p = Path(path)
    return parse_case(p.read_text(encoding="utf-8"), name=p.stem)


def write_case(case: RawCase) -> str:
    """Case text that :func:`parse_case` reads back bit-identically (%.17g);
    unconsumed MATPOWER columns are written as neutral placeholders."""
    g = lambda v: format(float(v), ".17g")
    out = [f"function mpc = {case.name or 'case'}", "mpc.version = '2';",
           f"mpc.baseMVA = {g(case.base_mva)};", "mpc.bus = ["]
    for i in range(case.n_bus):
        out.append(f"\t{int(case.bus_id[i])}\t{int(case.bus_type[i])}\t{g(case.pd[i])}"
                   f"\t{g(case.qd[i])}\t{g(case.gs[i])}\t{g(case.bs[i])}\t1\t{g(case.vm[i])}"
                   f"\t{g(case.va[i])}\t{g(case.base_kv[i])}\t1\t1.1\t0.9;")
    out += ["];", "mpc.gen = ["]
    for i in range(case.n_gen):
        out.append(f"\t{int(case.gen_bus[i])}\t{g(case.pg[i])}\t{g(case.qg[i])}"
                   f"\t{g(case.qmax[i])}\t{g(case.qmin[i])}\t{g(case.vg[i])}\t100"
                   f"\t{int(case.gen_status[i])}\t0\t0;")
    out += ["];", "mpc.branch = ["]
    for i in range(case.n_branch):
        out.append(f"\t{int(case.from_bus[i])}\t{int(case.to_bus[i])}\t{g(case.r[i])}"
                   f"\t{g(case.x[i])}\t{g(case.b[i])}\t0\t0\t0\t{g(case.ratio[i])}"
                   f"\t{g(case.angle[i])}\t{int(case.br_status[i])}\t-360\t360;")
    out.append("];")
    return "\n".join(out) + "\n"
