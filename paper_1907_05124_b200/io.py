"""Instance I/O and result documents -- the host-side mirror of include/mars/io.hpp
(src/io.cpp) around the B200 batch.

* G-set / rudy graphs: ``parse_gset`` (io.cpp:77-130), ``load_gset``, ``write_gset``
  (io.cpp:138-141), ``gset_to_problem`` (io.cpp:143-149; the 1-based -> 0-based shift happens
  here and nowhere else).
* Dense matrix text: ``read_matrix`` (io.cpp:187-222), ``write_matrix`` (io.cpp:165-178).
* ``detect_format`` (io.cpp:230-244), ``load_problem`` (io.cpp:246-258).
* ``problem_hash`` (io.cpp:260-290): FNV-1a of the canonical content, computed natively over
  the stored representation (C-ABI ``mars_problem_hash`` / ``mars_instance_hash``).
* Result documents: ``make_result_document`` (io.cpp:480-502),
  ``result_document_to_string`` / ``_from_string`` (io.cpp:504-592), ``save_result``,
  ``load_result``, ``verify_result_document`` (io.cpp:608-613).  The JSON text is the
  reference's byte for byte: nlohmann::json ``dump(2)`` -- sorted keys, two-space indent,
  shortest round-trip doubles with nlohmann's exponent thresholds -- plus a trailing newline.

Error classes and messages follow include/mars/errors.hpp and io.cpp.  Parsers run on the
host (they are not on the hot path); problems are created on the device through the C-ABI.
"""
from __future__ import annotations

import datetime
import enum
import json
import math
import re
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import mars as M
from ._native import lib, ptr


class ParseError(M.Error):
    """Malformed text input (errors.hpp: ParseError, 'line N: ' prefix when known)."""

    def __init__(self, msg: str, line: int = 0):
        super().__init__(f"line {line}: {msg}" if line else msg)
        self.line = line


class StructuralError(M.Error):
    """Parsed input violating a structural rule (edge counts, ranges, duplicates)."""


class IntegrityError(M.Error):
    """Document produced for a different problem."""


class VersionError(M.Error):
    """Document written by an incompatible format version."""


# ------------------------------------------------------------------ lexical helpers

_CSPACE = " \t\n\v\f\r"
_INT = re.compile(r"-?[0-9]+\Z")
_DEC = re.compile(r"[+-]?(?:[0-9]+\.?[0-9]*|\.[0-9]+)(?:[eE][+-]?[0-9]+)?\Z")
_HEX = re.compile(r"[+-]?0[xX](?:[0-9a-fA-F]+\.?[0-9a-fA-F]*|\.[0-9a-fA-F]+)(?:[pP][+-]?[0-9]+)?\Z")
_SPECIAL = re.compile(r"[+-]?(?:inf|infinity|nan(?:\([0-9A-Za-z_]*\))?)\Z", re.IGNORECASE)


def _lines(text: str):
    """std::getline over the text: pieces between '\\n' (a final empty piece is not a line)."""
    parts = text.split("\n")
    if parts and parts[-1] == "":
        parts.pop()
    return parts


def _comment_or_blank(line: str) -> bool:
    for c in line:
        if c in _CSPACE:
            continue
        return c in "#%"
    return True


def _tokens(line: str) -> List[str]:
    return [t for t in re.split(r"[ \t\n\v\f\r]+", line) if t]


def _int_token(tok: str, line: int, what: str) -> int:
    """std::from_chars<long long>: optional '-', decimal digits, whole token, in range."""
    if not _INT.match(tok):
        raise ParseError(f"expected integer {what}, got '{tok}'", line)
    v = int(tok)
    if not -(1 << 63) <= v < (1 << 63):
        raise ParseError(f"expected integer {what}, got '{tok}'", line)
    return v


def _as_int32(v: int) -> int:
    """static_cast<int>(long long): two's-complement truncation."""
    v &= 0xFFFFFFFF
    return v - (1 << 32) if v >= (1 << 31) else v


def _real_token(tok: str, line: int, what: str) -> float:
    """std::stod on the whole token (ERANGE -> out_of_range -> ParseError)."""
    err = ParseError(f"expected real {what}, got '{tok}'", line)
    if _SPECIAL.match(tok):
        return float(tok.split("(")[0])
    if _HEX.match(tok):
        body = tok.lstrip("+-")
        v = float.fromhex(body if "p" in body.lower() else body + "p0")
        v = -v if tok.startswith("-") else v
    elif _DEC.match(tok):
        v = float(tok)
    else:
        raise err
    if math.isinf(v):
        raise err                                  # overflow
    if v != 0.0 and abs(v) < 2.2250738585072014e-308:
        raise err                                  # underflow to a subnormal
    if v == 0.0 and re.search(r"[1-9]", tok.split("e")[0].split("E")[0].split("p")[0].split("P")[0]):
        raise err                                  # underflow to zero
    return v


# ------------------------------------------------------------------ G-set (io.hpp: GsetGraph)

@dataclass
class GsetEdge:
    u: int = 0          # 1-based, as in the file
    v: int = 0
    w: int = 1


@dataclass
class GsetGraph:
    n_vertices: int = 0
    edges: List[GsetEdge] = field(default_factory=list)


def parse_gset(text: str) -> GsetGraph:
    """io.cpp:77-130: header "n m", then m lines "u v [w]" (1-based, integer w, default 1)."""
    lines = _lines(text)
    g = GsetGraph()
    edge_count = -1
    pos = 0
    line_no = 0
    while pos < len(lines):
        line = lines[pos]
        pos += 1
        line_no += 1
        if _comment_or_blank(line):
            continue
        toks = _tokens(line)
        if len(toks) != 2:
            raise ParseError("header must be two integers: vertex count, edge count", line_no)
        g.n_vertices = _as_int32(_int_token(toks[0], line_no, "vertex count"))
        edge_count = _int_token(toks[1], line_no, "edge count")
        break
    if edge_count < 0:
        raise ParseError("missing header line")
    if g.n_vertices <= 0:
        raise StructuralError("vertex count must be positive")
    seen = set()
    while pos < len(lines):
        line = lines[pos]
        pos += 1
        line_no += 1
        if _comment_or_blank(line):
            continue
        toks = _tokens(line)
        if len(toks) not in (2, 3):
            raise ParseError("edge line must be 'u v' or 'u v w'", line_no)
        u = _as_int32(_int_token(toks[0], line_no, "endpoint"))
        v = _as_int32(_int_token(toks[1], line_no, "endpoint"))
        w = _int_token(toks[2], line_no, "weight") if len(toks) == 3 else 1
        n = g.n_vertices
        if u < 1 or u > n or v < 1 or v > n:
            raise StructuralError(f"line {line_no}: vertex out of range 1..{n}")
        if u == v:
            raise StructuralError(f"line {line_no}: self-loop at vertex {u}")
        key = (min(u, v) * 1000003 + max(u, v)) & 0xFFFFFFFFFFFFFFFF
        if key in seen:
            raise StructuralError(f"line {line_no}: duplicate edge ({u},{v})")
        seen.add(key)
        g.edges.append(GsetEdge(u, v, w))
        if len(g.edges) > edge_count:
            raise StructuralError(f"more edge lines than the declared count {edge_count}")
    if len(g.edges) != edge_count:
        raise StructuralError(f"edge count mismatch: header declares {edge_count}, file has {len(g.edges)}")
    return g


def _read_text(path: str) -> str:
    try:
        with open(path, "r", encoding="utf-8", errors="surrogateescape", newline="") as f:
            return f.read()
    except OSError:
        raise M.InputError(f"cannot open '{path}'") from None


def load_gset(path: str) -> GsetGraph:
    return parse_gset(_read_text(path))


def write_gset(g: GsetGraph) -> str:
    """io.cpp:138-141."""
    out = [f"{g.n_vertices} {len(g.edges)}\n"]
    out += [f"{e.u} {e.v} {e.w}\n" for e in g.edges]
    return "".join(out)


def gset_edges(g: GsetGraph):
    """The 0-based (u, v, w) arrays gset_to_problem hands to from_edges (io.cpp:143-149)."""
    u = np.array([e.u - 1 for e in g.edges], np.int32)
    v = np.array([e.v - 1 for e in g.edges], np.int32)
    w = np.array([float(e.w) for e in g.edges], np.float64)
    return u, v, w


def gset_to_problem(g: GsetGraph, device: int = 0, kernel: str = "auto") -> M.IsingProblem:
    """io.cpp:143-149: J_uv = J_vu = w, zero field, on the device."""
    p = M.IsingProblem.from_edges(g.n_vertices, gset_edges(g), device=device, kernel=kernel)
    p._host = ("edges", g.n_vertices, gset_edges(g), None)
    return p


# ------------------------------------------------------------------ dense matrix text

def parse_matrix(text: str) -> np.ndarray:
    """read_matrix (io.cpp:187-222) up to the IsingProblem::dense call: the n x n couplings,
    validated like IsingProblem::dense (errors re-raised as StructuralError, io.cpp:218-221)."""
    lines = _lines(text)
    n = -1
    pos = 0
    line_no = 0
    while pos < len(lines):
        line = lines[pos]
        pos += 1
        line_no += 1
        if _comment_or_blank(line):
            continue
        toks = _tokens(line)
        if len(toks) != 1:
            raise ParseError("matrix header must be a single integer n", line_no)
        n = _as_int32(_int_token(toks[0], line_no, "matrix size"))
        break
    if n <= 0:
        raise ParseError("missing or non-positive matrix size", line_no)
    J = np.zeros((n, n), np.float64)
    row = 0
    while row < n and pos < len(lines):
        line = lines[pos]
        pos += 1
        line_no += 1
        if _comment_or_blank(line):
            continue
        toks = _tokens(line)
        if len(toks) != n:
            raise ParseError(f"row {row} has {len(toks)} entries, expected {n}", line_no)
        J[row] = [_real_token(t, line_no, "entry") for t in toks]
        row += 1
    if row != n:
        raise ParseError(f"matrix ends after {row} of {n} rows")
    for i in range(n):                                                   # model.cpp:55-64
        if J[i, i] != 0.0:
            raise StructuralError(f"invalid matrix: coupling diagonal must be zero (row {i})")
        bad = np.nonzero(J[i, i + 1:] != J[i + 1:, i])[0]
        if bad.size:
            raise StructuralError(f"invalid matrix: coupling matrix must be symmetric (entries {i},{i + 1 + bad[0]})")
    return J


def read_matrix(text: str, device: int = 0, kernel: str = "auto") -> M.IsingProblem:
    J = parse_matrix(text)
    p = M.IsingProblem.dense(J.shape[0], J, device=device, kernel=kernel)
    p._host = ("dense", J.shape[0], J, None)
    return p


def read_matrix_file(path: str, device: int = 0, kernel: str = "auto") -> M.IsingProblem:
    return read_matrix(_read_text(path), device, kernel)


def _fmt17(v: float) -> str:
    """snprintf("%.17g") (io.cpp:57-61)."""
    return "%.17g" % v


def matrix_text(rows: np.ndarray) -> str:
    """write_matrix's text for the row_values of every row (io.cpp:165-178)."""
    n = rows.shape[0]
    out = [f"{n}\n"]
    for i in range(n):
        out.append(" ".join(_fmt17(x) for x in rows[i]) + "\n")
    return "".join(out)


def write_matrix(p: M.IsingProblem) -> str:
    """io.cpp:165-178: refused for problems with a nonzero field."""
    if p.has_field():
        raise M.InputError("the dense matrix format stores couplings only; field is nonzero")
    n = p.size()
    rows = np.zeros((n, n), np.float64)
    M._check(lib.mars_problem_rows(p._h, ptr(rows)))
    return matrix_text(rows)


class InstanceFormat(enum.Enum):
    GsetGraph = 0
    DenseMatrix = 1


def detect_format(text: str) -> InstanceFormat:
    """io.cpp:230-244: first data line of two tokens is a G-set header, one token a matrix."""
    for line_no, line in enumerate(_lines(text), 1):
        if _comment_or_blank(line):
            continue
        toks = _tokens(line)
        if len(toks) == 1:
            return InstanceFormat.DenseMatrix
        if len(toks) == 2:
            return InstanceFormat.GsetGraph
        raise ParseError(f"cannot detect format: first data line has {len(toks)} tokens (expected 1 or 2)",
                         line_no)
    raise ParseError("cannot detect format of an empty file")


@dataclass
class LoadedProblem:
    problem: M.IsingProblem
    format: InstanceFormat


def load_problem(path: str, forced: Optional[InstanceFormat] = None, device: int = 0,
                 kernel: str = "auto") -> LoadedProblem:
    """io.cpp:246-258, creating the problem on `device`."""
    text = _read_text(path)
    fmt = forced if forced is not None else detect_format(text)
    if fmt == InstanceFormat.GsetGraph:
        return LoadedProblem(gset_to_problem(parse_gset(text), device, kernel), fmt)
    return LoadedProblem(read_matrix(text, device, kernel), fmt)


# ------------------------------------------------------------------ problem_hash

def instance_hash(n: int, J=None, edges=None, field=None) -> int:
    """problem_hash of an instance given as dense J or (u, v, w) edges, without a device
    (same validation and storage rule as the constructors; C-ABI mars_instance_hash)."""
    out = np.zeros(1, np.uint64)
    h = None if field is None else np.ascontiguousarray(field, np.float64)
    if J is not None:
        Jc = np.ascontiguousarray(J, np.float64).reshape(-1)
        M._check(lib.mars_instance_hash(int(n), ptr(Jc), 0, None, None, None, ptr(h), ptr(out)))
    else:
        u, v, w = (np.ascontiguousarray(edges[0], np.int32), np.ascontiguousarray(edges[1], np.int32),
                   np.ascontiguousarray(edges[2], np.float64))
        M._check(lib.mars_instance_hash(int(n), None, len(u), ptr(u), ptr(v), ptr(w), ptr(h), ptr(out)))
    return int(out[0])


@dataclass
class HostInstance:
    """An instance described on the host only (dense J or (u, v, w) edges, optional field):
    enough for problem_hash and result documents without a device."""
    n: int
    J: Optional[np.ndarray] = None
    edges: Optional[tuple] = None
    field: Optional[np.ndarray] = None

    def size(self) -> int:
        return self.n


def problem_hash(p) -> int:
    """io.cpp:260-290 over the problem's stored representation (device IsingProblem or
    HostInstance)."""
    if isinstance(p, HostInstance):
        return instance_hash(p.n, p.J, p.edges, p.field)
    out = np.zeros(1, np.uint64)
    M._check(lib.mars_problem_hash(p._h, ptr(out)))
    return int(out[0])


def hash_to_hex(h: int) -> str:
    return "%016x" % (h & 0xFFFFFFFFFFFFFFFF)


def hash_from_hex(s: str) -> int:
    h = 0
    for c in s:
        if "0" <= c <= "9" or "a" <= c <= "f":
            h = ((h << 4) | int(c, 16)) & 0xFFFFFFFFFFFFFFFF
        else:
            raise ParseError("invalid hash digit in document")
    return h


# ------------------------------------------------------------------ result documents

kResultDocVersion = 1


class DocDetail(enum.IntEnum):
    Summary = 0
    Energies = 1
    Full = 2


@dataclass
class ResultDocument:
    """io.hpp: ResultDocument."""
    version: int = kResultDocVersion
    problem_id: str = ""
    problem_hash: int = 0
    problem_size: int = 0
    solver: str = "mars"
    params: M.MarsParams = field(default_factory=M.MarsParams)
    stats: M.BatchStats = field(default_factory=M.BatchStats)
    runs: List[M.RunResult] = field(default_factory=list)
    detail: DocDetail = DocDetail.Energies
    include_volatile: bool = True
    timestamp: str = ""


def _iso_now() -> str:
    return datetime.datetime.now(datetime.timezone.utc).strftime("%Y-%m-%dT%H:%M:%SZ")


def make_result_document(problem_id: str, problem, params: M.MarsParams,
                         stats: M.BatchStats, detail: DocDetail = DocDetail.Full,
                         include_volatile: bool = True) -> ResultDocument:
    """io.cpp:480-502 (`problem`: IsingProblem or HostInstance).  A Full document needs every
    run's spins: run the batch with ``BatchSpec(keep_spins=True)``."""
    runs = stats.runs if detail == DocDetail.Full else []
    if detail == DocDetail.Full and stats.records is not None and stats.records.spins is None:
        raise M.InputError("a full result document needs the batch's spins (BatchSpec.keep_spins=True)")
    s = M.BatchStats(stats.best_energy, stats.mean_energy, stats.best_cut, stats.mean_cut, stats.hit_count,
                     stats.success_probability, stats.total_seconds, stats.mean_seconds_per_run,
                     M.RunResult(**vars(stats.best_result)), np.asarray(stats.energies).copy(),
                     stats.completed_runs, stats.skipped_runs, stats.failed_runs)
    if detail == DocDetail.Summary:
        s.energies = np.zeros(0)
    if not include_volatile:
        s.total_seconds = 0.0
        s.mean_seconds_per_run = 0.0
        s.best_result.elapsed_seconds = 0.0
        for r in runs:
            r.elapsed_seconds = 0.0
    return ResultDocument(kResultDocVersion, problem_id, problem_hash(problem), problem.size(), "mars",
                          params, s, runs, detail, include_volatile,
                          _iso_now() if include_volatile else "")


class _Real(float):
    """A double that json.dumps writes the way nlohmann::json's dump does."""

    def __repr__(self):
        return _nlohmann_double(float(self))


def _nlohmann_double(v: float) -> str:
    """nlohmann::detail::to_chars: shortest round-trip digits d1..dk with decimal exponent n
    (value = 0.d1..dk x 10^n); plain notation for -4 < n <= 15, else d1.d2..dk e+XX."""
    if math.isnan(v) or math.isinf(v):
        return "null"
    if v == 0.0:
        return "-0.0" if math.copysign(1.0, v) < 0 else "0.0"
    sign = "-" if v < 0 else ""
    digits, exp = repr(abs(v)).lower().split("e") if "e" in repr(abs(v)).lower() else (repr(abs(v)), "0")
    intpart, _, frac = digits.partition(".")
    mant = (intpart + frac).lstrip("0")
    point = len(intpart) + int(exp) if intpart != "0" else int(exp) - (len(frac) - len(frac.lstrip("0")))
    mant = mant.rstrip("0") or "0"
    k, n = len(mant), point
    if k <= n <= 15:
        return sign + mant + "0" * (n - k) + ".0"
    if 0 < n <= 15:
        return sign + mant[:n] + "." + mant[n:]
    if -4 < n <= 0:
        return sign + "0." + "0" * (-n) + mant
    e = n - 1
    body = mant[0] + ("." + mant[1:] if k > 1 else "")
    return sign + body + "e" + ("-" if e < 0 else "+") + "%02d" % abs(e)


def _spins_str(spins) -> str:
    return "".join("+" if x > 0 else "-" for x in np.asarray(spins))


_STATUS = {M.RunStatus.Ok: "ok", M.RunStatus.Skipped: "skipped", M.RunStatus.Diverged: "diverged"}


def _run_json(r: M.RunResult, include_volatile: bool) -> dict:
    j = {"status": _STATUS[M.RunStatus(r.status)], "start_temp": _Real(r.start_temp)}
    if r.status != M.RunStatus.Skipped:
        j["energy"] = _Real(r.energy)
        j["cut"] = _Real(r.cut)
        j["descent_iters"] = int(r.descent_iters)
        j["spins"] = _spins_str(r.spins) if r.spins is not None else ""
        if include_volatile:
            j["elapsed_seconds"] = _Real(r.elapsed_seconds)
    if r.error:
        j["error"] = r.error
    return j


def _params_json(p: M.MarsParams) -> dict:
    """solver_params_to_json for MarsParams (io.cpp:295-302)."""
    return {"t_min": _Real(p.t_min), "t_max": _Real(p.t_max), "t_step": _Real(p.t_step),
            "c_step": _Real(p.c_step), "d_min": _Real(p.d_min),
            "start_mode": "grid" if p.start_mode == M.StartMode.GridSweep else "random"}


def result_document_to_string(doc: ResultDocument) -> str:
    """io.cpp:504-538."""
    j = {"format": "mars-result", "version": doc.version}
    if doc.include_volatile:
        j["created"] = doc.timestamp
    j["problem"] = {"id": doc.problem_id, "hash": hash_to_hex(doc.problem_hash), "n": doc.problem_size}
    j["solver"] = {"name": doc.solver, "params": _params_json(doc.params)}
    st = doc.stats
    s = {"best_energy": _Real(st.best_energy), "mean_energy": _Real(st.mean_energy),
         "best_cut": _Real(st.best_cut), "mean_cut": _Real(st.mean_cut), "hit_count": int(st.hit_count),
         "success_probability": _Real(st.success_probability), "completed_runs": int(st.completed_runs),
         "skipped_runs": int(st.skipped_runs), "failed_runs": int(st.failed_runs)}
    if doc.include_volatile:
        s["total_seconds"] = _Real(st.total_seconds)
        s["mean_seconds_per_run"] = _Real(st.mean_seconds_per_run)
    if doc.detail != DocDetail.Summary:
        s["energies"] = [_Real(x) for x in np.asarray(st.energies, np.float64)]
    s["best_run"] = _run_json(st.best_result, doc.include_volatile)
    j["stats"] = s
    if doc.detail == DocDetail.Full:
        j["runs"] = [_run_json(r, doc.include_volatile) for r in doc.runs]
    return _dump(j) + "\n"


def _dump(obj, indent: int = 0) -> str:
    """nlohmann::json::dump(2) (sorted object keys, ', ' never used, empty [] / {})."""
    pad = " " * (indent + 2)
    if isinstance(obj, dict):
        if not obj:
            return "{}"
        items = [f'{pad}{json.dumps(k, ensure_ascii=False)}: {_dump(obj[k], indent + 2)}' for k in sorted(obj)]
        return "{\n" + ",\n".join(items) + "\n" + " " * indent + "}"
    if isinstance(obj, list):
        if not obj:
            return "[]"
        return "[\n" + ",\n".join(pad + _dump(x, indent + 2) for x in obj) + "\n" + " " * indent + "]"
    if isinstance(obj, _Real):
        return repr(obj)
    if isinstance(obj, bool):
        return "true" if obj else "false"
    if isinstance(obj, int):
        return str(obj)
    if isinstance(obj, float):
        return _nlohmann_double(obj)
    return json.dumps(obj, ensure_ascii=False)


def result_document_from_string(text: str) -> ResultDocument:
    """io.cpp:540-592."""
    try:
        j = json.loads(text)
    except ValueError as e:
        raise ParseError(f"invalid result document: {e}") from None
    try:
        if j.get("format", "") != "mars-result":
            raise ParseError("not a mars-result document")
        doc = ResultDocument()
        doc.version = int(j["version"])
        if doc.version != kResultDocVersion:
            raise VersionError(f"result document version {doc.version} is not supported "
                               f"(expected {kResultDocVersion})")
        doc.include_volatile = "created" in j
        doc.timestamp = j["created"] if doc.include_volatile else ""
        doc.problem_id = j["problem"]["id"]
        doc.problem_hash = hash_from_hex(j["problem"]["hash"])
        doc.problem_size = int(j["problem"]["n"])
        doc.solver = j["solver"]["name"]
        if doc.solver != "mars":
            raise ParseError(f"unknown solver '{doc.solver}' in result document")
        pj = j["solver"]["params"]
        doc.params = M.MarsParams(pj["t_min"], pj["t_max"], pj["t_step"], pj["c_step"], pj["d_min"],
                                  M.StartMode.GridSweep if pj["start_mode"] == "grid" else M.StartMode.UniformRandom)
        s = j["stats"]
        st = M.BatchStats(s["best_energy"], s["mean_energy"], s["best_cut"], s["mean_cut"], int(s["hit_count"]),
                          s["success_probability"], s.get("total_seconds", 0.0), s.get("mean_seconds_per_run", 0.0))
        st.completed_runs, st.skipped_runs, st.failed_runs = (int(s["completed_runs"]), int(s["skipped_runs"]),
                                                               int(s["failed_runs"]))
        st.energies = np.asarray(s.get("energies", []), np.float64)
        st.best_result = _run_from(s["best_run"])
        doc.stats = st
        if "runs" in j:
            doc.detail = DocDetail.Full
            doc.runs = [_run_from(r) for r in j["runs"]]
        else:
            doc.detail = DocDetail.Energies if "energies" in s else DocDetail.Summary
        return doc
    except (KeyError, TypeError) as e:
        raise ParseError(f"malformed result document: {e}") from None


def _run_from(j: dict) -> M.RunResult:
    names = {v: k for k, v in _STATUS.items()}
    if j["status"] not in names:
        raise ParseError(f"invalid run status '{j['status']}'")
    r = M.RunResult(names[j["status"]], start_temp=j["start_temp"])
    if r.status != M.RunStatus.Skipped:
        r.energy, r.cut, r.descent_iters = j["energy"], j["cut"], int(j["descent_iters"])
        s = j["spins"]
        if any(c not in "+-" for c in s):
            raise ParseError("invalid spin character in document")
        r.spins = np.array([1 if c == "+" else -1 for c in s], np.int8)
        r.elapsed_seconds = j.get("elapsed_seconds", 0.0)
    r.error = j.get("error", "")
    return r


def save_result(doc: ResultDocument, path: str) -> None:
    try:
        with open(path, "w", encoding="utf-8", newline="") as f:
            f.write(result_document_to_string(doc))
    except OSError:
        raise M.InputError(f"cannot write '{path}'") from None


def load_result(path: str) -> ResultDocument:
    return result_document_from_string(_read_text(path))


def verify_result_document(doc: ResultDocument, p) -> None:
    """io.cpp:608-613."""
    h = problem_hash(p)
    if doc.problem_hash != h or doc.problem_size != p.size():
        raise IntegrityError(f"result document was produced for a different problem (hash "
                             f"{hash_to_hex(doc.problem_hash)} vs {hash_to_hex(h)})")
