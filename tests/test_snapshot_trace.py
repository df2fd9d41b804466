"""SDC1 field snapshots and PMISDC schedule traces against the unmodified reference (CPU).

  write_field_snapshot / read_field_snapshot   reaction_diffusion.cpp:230-259
  build_task_graph / validate_schedule_trace / write_trace_csv   pipeline.cpp:36-70, 322-361
The GPU side of the trace (a real two-stream sweep) is in test_gpu_parity.py.
"""
import numpy as np
import pytest

from paper_1801_01201_b200 import api


def test_snapshot_bytes_equal_reference(tmp_path, ref):
    rng = np.random.default_rng(3)
    data = rng.standard_normal(257)
    ours, theirs = tmp_path / "a.sdc", tmp_path / "b.sdc"
    api.write_field_snapshot(str(ours), 257, 0.078125, data)
    ref.ref_write_field_snapshot(str(theirs), 257, 0.078125, data)
    assert ours.read_bytes() == theirs.read_bytes()
    n, dx, back = ref.ref_read_field_snapshot(str(ours))
    assert n == 257 and dx == 0.078125 and np.array_equal(back, data)
    s = api.read_field_snapshot(str(theirs))
    assert s.n_x == 257 and s.dx == 0.078125 and np.array_equal(s.data, data)


def test_snapshot_empty_and_errors(tmp_path, ref):
    p = tmp_path / "e.sdc"
    api.write_field_snapshot(str(p), 0, 1.0, np.empty(0))
    s = api.read_field_snapshot(str(p))
    assert s.n_x == 0 and s.data.size == 0
    with pytest.raises(ValueError, match="write_field_snapshot: size mismatch"):
        api.write_field_snapshot(str(p), 5, 1.0, np.zeros(4))
    with pytest.raises(RuntimeError, match="read_field_snapshot: cannot open"):
        api.read_field_snapshot(str(tmp_path / "missing.sdc"))
    bad = tmp_path / "bad.sdc"
    bad.write_bytes(b"SDC2" + b"\0" * 12)
    with pytest.raises(RuntimeError, match="read_field_snapshot: bad magic"):
        api.read_field_snapshot(str(bad))
    trunc = tmp_path / "t.sdc"
    api.write_field_snapshot(str(trunc), 8, 0.5, np.arange(8.0))
    trunc.write_bytes(trunc.read_bytes()[:-3])
    with pytest.raises(RuntimeError, match="read_field_snapshot: truncated file"):
        api.read_field_snapshot(str(trunc))
    with pytest.raises(Exception, match="truncated"):
        ref.ref_read_field_snapshot(str(trunc))
    with pytest.raises(RuntimeError, match="write_field_snapshot: cannot open"):
        api.write_field_snapshot(str(tmp_path / "no" / "dir.sdc"), 1, 1.0, np.zeros(1))


def serial_trace(M, nu, workers=2, gap=0):
    """A trace of the serial cell order (D, R alternating, one cell at a time)."""
    g = api.build_task_graph(M, nu)
    cells = [None] * len(g.cells)
    t, seq = 0, 0
    for ell in range(1, nu + 1):
        for m in range(1, M + 1):
            for kind in (api.CellKind.diffusion, api.CellKind.reaction):
                i = g.cell_id(kind, m, ell)
                cells[i] = api.CellTrace(g.cells[i], int(kind) % workers, t, t + 10, seq, seq + 1)
                t += 10 + gap
                seq += 2
    return g, api.ScheduleTrace(workers, cells)


@pytest.mark.parametrize("M,nu", [(2, 1), (4, 3), (6, 1), (3, 8)])
def test_task_graph_and_validator_match_reference(ref, M, nu):
    g, tr = serial_trace(M, nu)
    assert api.validate_schedule_trace(g, tr) == ""
    assert ref.ref_validate_schedule_trace(M, nu, tr) == ""
    # break every edge in turn: both validators must name the same violation
    for v in range(len(g.cells)):
        for u in g.dependencies[v]:
            cells = list(tr.cells)
            a, b = cells[u], cells[v]
            cells[v] = api.CellTrace(b.cell, b.worker, a.end_ns - 1, b.end_ns, b.seq_start, b.seq_end)
            bad = api.ScheduleTrace(tr.workers, cells)
            ours = api.validate_schedule_trace(g, bad)
            assert ours.startswith("edge violated") or ours.startswith("worker overlap")
            assert ours == ref.ref_validate_schedule_trace(M, nu, bad)


def test_trace_csv_schema():
    """write_trace_csv (pipeline.cpp:352-361): header and one row per cell in cell-id order.  (The
    reference's own writer is not called in-process: its formatted-stream output crashes when the
    statically linked C++ runtime of oracle/_ref meets the interpreter's; the schema is fixed text.)"""
    _, tr = serial_trace(2, 1)
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        p = d + "/t.csv"
        api.write_trace_csv(p, tr)
        text = open(p).read()
    assert text == ("cell,kind,m,ell,worker,start_ns,end_ns\n"
                    "D(1,1),D,1,1,0,0,10\nR(1,1),R,1,1,1,10,20\nD(2,1),D,2,1,0,20,30\nR(2,1),R,2,1,1,30,40\n")
