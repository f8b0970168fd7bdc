"""Scenario and trajectory I/O.

* The reference's text format (``FAST-SCENARIO v1``, world.hpp:267-399): `parse_scenario`,
  `serialize_scenario`, `load_scenario` -- same grammar, same line-numbered errors.  It costs a
  character per cell and parses serially, so for ≥ 1e8-cell grids there is also
* a binary format (``FASTSCB1``): a 40-byte little-endian header (magic, width, height,
  cell_size, boundary, flags) then the CellKind bytes row-major and, optionally, the fp64 static
  field -- read back with one `numpy.fromfile` per array (memory-mappable), so a plaza loads in
  well under a second and the field need not be recomputed.
* A trajectory / occupancy dump (``FASTTRJ1``) mirroring the acceptance tests' `StepSnapshot`
  (positions, alive bits, exit ids in processing order; tests/acceptance.cpp:46-73), optionally
  with the occupancy grid (cell -> agent id or -1, the reference's i32 layout) per frame.
"""
from __future__ import annotations

import os
import re
import struct
from dataclasses import dataclass
from typing import Iterator, List, Optional

import numpy as np

from . import fastped as fp

SCENARIO_HEADER = "FAST-SCENARIO v1"
BINARY_MAGIC = b"FASTSCB1"
TRAJ_MAGIC = b"FASTTRJ1"
_CHAR = {"#": fp.WALL, ".": fp.FREE, "E": fp.EXIT}
_GLYPH = np.array([".", "#", "E"])  # indexed by CellKind


def _scenario_error(line: int, msg: str):
    raise RuntimeError("scenario line %d: %s" % (line, msg))  # detail::scenario_error (world.hpp:269-271)


def _split_lines(text: str) -> List[str]:
    """detail::split_lines (world.hpp:273-286): '\\n' separated, a trailing '\\r' dropped."""
    return [ln[:-1] if ln.endswith("\r") else ln for ln in text.split("\n")]


_INT = re.compile(r"-?[0-9]+\Z")
_FLOAT = re.compile(r"-?(?:[0-9]+\.?[0-9]*|\.[0-9]+)(?:[eE][-+]?[0-9]+)?\Z|-?(?:inf|infinity|nan)\Z", re.I)


def _parse_field(line: str, line_no: int, key: str, kind):
    """detail::parse_field (world.hpp:288-302): '<key> <value>', the value in from_chars form."""
    if not line.startswith(key) or len(line) <= len(key) or line[len(key)] != " ":
        _scenario_error(line_no, "expected '%s <value>'" % key)
    value = line[len(key) + 1:]
    if not (_INT if kind is int else _FLOAT).match(value):
        _scenario_error(line_no, "malformed value for '%s'" % key)
    return kind(value)


def parse_scenario(text: str) -> fp.Grid:
    """parse_scenario (world.hpp:304-370)."""
    lines = _split_lines(text)

    def line_at(i):
        return lines[i] if i < len(lines) else ""

    if line_at(0) != SCENARIO_HEADER:
        _scenario_error(1, "malformed header, expected '%s'" % SCENARIO_HEADER)
    width = _parse_field(line_at(1), 2, "width", int)
    height = _parse_field(line_at(2), 3, "height", int)
    cell_size = _parse_field(line_at(3), 4, "cell_size", float)
    if width < 1:
        _scenario_error(2, "width must be >= 1")
    if height < 1:
        _scenario_error(3, "height must be >= 1")
    if not cell_size > 0.0:
        _scenario_error(4, "cell_size must be > 0")
    if line_at(4) == "boundary closed":
        boundary = fp.CLOSED
    elif line_at(4) == "boundary periodic-x":
        boundary = fp.PERIODIC_X
    else:
        _scenario_error(5, "expected 'boundary closed' or 'boundary periodic-x'")
    if line_at(5) != "grid:":
        _scenario_error(6, "expected 'grid:'")
    cells = np.empty((height, width), np.uint8)
    for y in range(height):
        li = 6 + y
        line_no = li + 1
        if li >= len(lines):
            _scenario_error(line_no, "dimension mismatch: expected %d grid rows, found %d" % (height, y))
        row = lines[li]
        if len(row) != width:
            _scenario_error(line_no, "dimension mismatch: row has %d cells, expected %d" % (len(row), width))
        for x, ch in enumerate(row):
            k = _CHAR.get(ch)
            if k is None:
                _scenario_error(line_no, "unknown cell character '%s'" % ch)
            cells[y, x] = k
    for li in range(6 + height, len(lines)):
        if lines[li]:
            _scenario_error(li + 1, "dimension mismatch: unexpected content after grid body")
    # boundary legality, reported with the line number (world.hpp:349-367)
    for y in range(height):
        for x in range(width):
            k = cells[y, x]
            if boundary == fp.CLOSED:
                if (y == 0 or y == height - 1 or x == 0 or x == width - 1) and k == fp.FREE:
                    _scenario_error(7 + y, "closed boundary violated: border cell at column %d must be '#' or 'E'" % x)
            elif (y == 0 or y == height - 1) and k != fp.WALL:
                _scenario_error(7 + y, "periodic-x boundary violated: top and bottom rows must be '#' (column %d)" % x)
    return fp.Grid(cells, cell_size, boundary)


def serialize_scenario(g: fp.Grid) -> str:
    """serialize_scenario (world.hpp:372-399); cell_size in shortest round-trip form."""
    head = "%s\nwidth %d\nheight %d\ncell_size %s\n%s\ngrid:\n" % (
        SCENARIO_HEADER, g.width, g.height, repr(float(g.cell_size)),
        "boundary closed" if g.boundary == fp.CLOSED else "boundary periodic-x")
    body = "\n".join("".join(r) for r in _GLYPH[g.cells]) + "\n"
    return head + body


def load_scenario(path: str, device: int = 0) -> fp.Scenario:
    """load_scenario (scenario_io.hpp:33-39): the file name is the scenario name; the field is
    computed on the device."""
    try:
        with open(path, "rb") as f:
            text = f.read().decode()
    except OSError:
        raise RuntimeError("cannot open scenario file: " + str(path)) from None
    return fp.make_scenario(os.path.basename(path), parse_scenario(text), device)


def save_scenario(g: fp.Grid, path: str):
    """write_text_file(serialize_scenario(g)) (scenario_io.hpp:179-186)."""
    with open(path, "wb") as f:
        f.write(serialize_scenario(g).encode())


# ---------------------------------------------------------------------------------- binary scenarios
_BIN_HEAD = struct.Struct("<8sqqdii")  # magic, width, height, cell_size, boundary, flags (bit 0: field)


def save_scenario_binary(sc_or_grid, path: str, with_field: bool = True):
    """Binary scenario: header, CellKind bytes (row-major), then the fp64 field when present."""
    g = sc_or_grid.grid if isinstance(sc_or_grid, fp.Scenario) else sc_or_grid
    field = sc_or_grid.field if (with_field and isinstance(sc_or_grid, fp.Scenario)) else None
    with open(path, "wb") as f:
        f.write(_BIN_HEAD.pack(BINARY_MAGIC, g.width, g.height, float(g.cell_size), int(g.boundary),
                               1 if field is not None else 0))
        np.ascontiguousarray(g.cells, np.uint8).tofile(f)
        if field is not None:
            np.ascontiguousarray(field, np.float64).reshape(g.height, g.width).tofile(f)


def load_scenario_binary(path: str, name: Optional[str] = None, device: int = 0) -> fp.Scenario:
    """Reads save_scenario_binary's file; recomputes the field on the device only if absent."""
    with open(path, "rb") as f:
        head = f.read(_BIN_HEAD.size)
        if len(head) != _BIN_HEAD.size:
            raise RuntimeError("binary scenario: truncated header: " + str(path))
        magic, w, h, cell, boundary, flags = _BIN_HEAD.unpack(head)
        if magic != BINARY_MAGIC:
            raise RuntimeError("binary scenario: bad magic in " + str(path))
        if w < 1 or h < 1:
            raise RuntimeError("binary scenario: bad dimensions %dx%d" % (w, h))
        cells = np.fromfile(f, np.uint8, w * h)
        if cells.size != w * h:
            raise RuntimeError("binary scenario: truncated cell data")
        field = None
        if flags & 1:
            field = np.fromfile(f, np.float64, w * h)
            if field.size != w * h:
                raise RuntimeError("binary scenario: truncated field data")
            field = field.reshape(h, w)
    g = fp.Grid(cells.reshape(h, w), cell, boundary)
    if field is None:
        field = fp.compute_static_field(g, device)
    return fp.Scenario(name or os.path.basename(path), g, field)


# ---------------------------------------------------------------------------------- trajectories
@dataclass
class StepSnapshot:
    """tests/acceptance.cpp:46-51 (+ the step index and, optionally, the occupancy grid)."""
    step: int
    x: np.ndarray          # int32 per agent
    y: np.ndarray          # int32 per agent
    alive: np.ndarray      # bool per agent
    exited: np.ndarray     # uint32 ids, processing order
    occupancy: Optional[np.ndarray] = None  # int32 HxW: agent id or -1

    def __eq__(self, o):
        same_occ = (self.occupancy is None) == (o.occupancy is None) and (
            self.occupancy is None or np.array_equal(self.occupancy, o.occupancy))
        return (self.step == o.step and np.array_equal(self.x, o.x) and np.array_equal(self.y, o.y) and
                np.array_equal(self.alive, o.alive) and np.array_equal(self.exited, o.exited) and same_occ)


_TRAJ_HEAD = struct.Struct("<8sqiii")  # magic, agents, width, height, flags (bit 0: occupancy)
_FRAME_HEAD = struct.Struct("<qq")     # step, exits


class TrajectoryWriter:
    """Appends frames: step, x, y (int32 each), alive (bit-packed), exit ids, [occupancy int32]."""

    def __init__(self, path: str, n_agents: int, width: int, height: int, with_occupancy: bool = False):
        self.n, self.w, self.h, self.occ = n_agents, width, height, with_occupancy
        self.f = open(path, "wb")
        self.f.write(_TRAJ_HEAD.pack(TRAJ_MAGIC, n_agents, width, height, 1 if with_occupancy else 0))

    def write(self, snap: StepSnapshot):
        ex = np.ascontiguousarray(snap.exited, np.uint32)
        self.f.write(_FRAME_HEAD.pack(int(snap.step), ex.size))
        np.ascontiguousarray(snap.x, np.int32).tofile(self.f)
        np.ascontiguousarray(snap.y, np.int32).tofile(self.f)
        np.packbits(np.asarray(snap.alive, bool)).tofile(self.f)
        ex.tofile(self.f)
        if self.occ:
            if snap.occupancy is None:
                raise ValueError("trajectory: this file carries occupancy frames")
            np.ascontiguousarray(snap.occupancy, np.int32).tofile(self.f)

    def close(self):
        self.f.close()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


def read_trajectory(path: str) -> Iterator[StepSnapshot]:
    with open(path, "rb") as f:
        head = f.read(_TRAJ_HEAD.size)
        magic, n, w, h, flags = _TRAJ_HEAD.unpack(head)
        if magic != TRAJ_MAGIC:
            raise RuntimeError("trajectory: bad magic in " + str(path))
        while True:
            fh = f.read(_FRAME_HEAD.size)
            if not fh:
                return
            step, ne = _FRAME_HEAD.unpack(fh)
            x = np.fromfile(f, np.int32, n)
            y = np.fromfile(f, np.int32, n)
            alive = np.unpackbits(np.fromfile(f, np.uint8, (n + 7) // 8), count=n).astype(bool)
            ex = np.fromfile(f, np.uint32, ne)
            occ = np.fromfile(f, np.int32, w * h).reshape(h, w) if flags & 1 else None
            yield StepSnapshot(step, x, y, alive, ex, occ)


def snapshot(st: fp.SimState, exited, with_occupancy: bool = False) -> StepSnapshot:
    x, y, a = st.agents()
    return StepSnapshot(st.step, x.copy(), y.copy(), a.astype(bool), np.asarray(exited, np.uint32),
                        st.occupancy() if with_occupancy else None)


def record_trajectory(sc: fp.Scenario, agents: int, params: fp.SimParams, cores: int, steps: int,
                      path: Optional[str] = None, with_occupancy: bool = False,
                      device: int = 0) -> List[StepSnapshot]:
    """record_trajectory (tests/acceptance.cpp:53-73) on the device: plan_phase + move_phase +
    ++step per step, one snapshot per step; optionally streamed to a trajectory file."""
    st = fp.make_state(sc, fp.spawn_agents(sc.grid, agents, params.v_max, params.seed), device=device)
    out = []
    w = TrajectoryWriter(path, agents, sc.grid.width, sc.grid.height, with_occupancy) if path else None
    try:
        for _ in range(steps):
            fp.plan_phase(st, params, fp.ScheduleParams(cores))
            mv = fp.move_phase(st, params)
            st.step = st.step + 1
            snap = snapshot(st, mv.exited, with_occupancy)
            out.append(snap)
            if w:
                w.write(snap)
    finally:
        if w:
            w.close()
        st.close()
    return out
