"""On-disk datasets: the reference's text layout and the
binary twin, checked against the compiled reference's own save_dataset /
load_dataset (src/dataset_io.cpp:40-165, oracle/_ref).

CPU tests drive the host-side reader / writer through the C ABI (no GPU);
GPU tests load into / save from the HBM graph store."""
import filecmp
import os

import numpy as np
import pytest

SMALL = dict(n=300, avg_degree=4, dim=8, T=6, edge=0.05, feat=0.05)


@pytest.fixture(scope="module")
def api():
    from paper_2501_15348_b200 import api as A
    return A


def _ref_graph(ref, seed=1):
    s = SMALL
    return ref.RefGraph.synth(s["n"], s["avg_degree"], s["dim"], s["T"], s["edge"], s["feat"], seed=seed)


def _synth(api, seed=1):
    s = SMALL
    return api.Synth(s["n"], s["avg_degree"], s["dim"], s["T"], s["edge"], s["feat"], seed=seed)


def _read_all(api, path):
    ds = api.Dataset(path)
    return ds, ds.base(), [ds.step(t) for t in range(1, ds.T)]


def test_text_reader_matches_reference_loader(ref, api, tmp_path):
    """Reference-written text dataset: our reader yields exactly what the
    reference's loader reads (edges bitwise, features = fp32 of its stod)."""
    g = _ref_graph(ref)
    g.save_dataset(tmp_path)
    L = ref.RefGraph.load_dataset(tmp_path)
    ds, (src, dst, feats), steps = _read_all(api, tmp_path)
    assert (ds.num_nodes, ds.feature_dim, ds.T, ds.format) == (g.n, g.dim, g.T, 1)
    rs, rd = L.edges(0)
    assert np.array_equal(src, rs) and np.array_equal(dst, rd)
    assert np.array_equal(feats, L.feats(0).astype(np.float32))
    for t, st in enumerate(steps, start=1):
        d = g.delta(t)  # what the writer wrote
        for k in ("del_src", "del_dst", "ins_src", "ins_dst", "changed"):
            assert np.array_equal(st[k], d[k]), (t, k)
        ft = L.feats(t)[st["changed"]].astype(np.float32)
        assert np.array_equal(st["changed_feats"], ft), t


def test_text_writer_is_reference_fixed_point(ref, api, tmp_path):
    """Our text writer's manifest and snapshot_0 files are byte-identical to
    what the reference writes after loading them (load -> save idempotence),
    and snapshot_0.edges matches the reference writer on the same graph."""
    s = _synth(api)
    ours, again, theirs = tmp_path / "ours", tmp_path / "again", tmp_path / "theirs"
    s.save(ours, binary=False)
    ref.RefGraph.load_dataset(ours).save_dataset(again)
    _ref_graph(ref).save_dataset(theirs)
    for f in ("manifest.json", "snapshot_0.edges", "snapshot_0.feats"):
        assert filecmp.cmp(ours / f, again / f, shallow=False), f
    for f in ("manifest.json", "snapshot_0.edges"):
        assert filecmp.cmp(ours / f, theirs / f, shallow=False), f


@pytest.mark.parametrize("binary", [True, False])
def test_compact_round_trip(api, tmp_path, binary):
    s = _synth(api)
    s.save(tmp_path, binary=binary)
    ds, (src, dst, feats), steps = _read_all(api, tmp_path)
    assert ds.format == (2 if binary else 1)
    s0, d0, f0 = s.base()
    assert np.array_equal(src, s0) and np.array_equal(dst, d0) and np.array_equal(feats, f0)
    for t, st in enumerate(steps, start=1):
        want = s.step(t)
        for k in want:
            assert np.array_equal(st[k], want[k]), (t, k)


def _write(p, name, text):
    os.makedirs(p, exist_ok=True)
    with open(os.path.join(p, name), "w") as f:
        f.write(text)


def _tiny(p, edges="0\t1\n1\t2\n", feats="0.5,1\n-1,2\n3,4\n", d_edges="D 0 1\nI 2 0\n",
          d_feats="1,7,8\n", manifest='{"T":2,"feature_dim":2,"format_version":1,"num_nodes":3}\n'):
    _write(p, "manifest.json", manifest)
    _write(p, "snapshot_0.edges", edges)
    _write(p, "snapshot_0.feats", feats)
    _write(p, "delta_1.edges", d_edges)
    _write(p, "delta_1.feats", d_feats)
    return p


MALFORMED = {
    "bad_tag": dict(d_edges="D 0 1\nX 2 0\n"),
    "arity": dict(d_feats="1,7\n"),
    "feats_truncated": dict(feats="0.5,1\n-1,2\n"),
    "row_truncated": dict(feats="0.5,1\n-1\n3,4\n"),
    "empty_row": dict(feats="0.5,1\n\n3,4\n"),
    "bad_number": dict(feats="0.5,1\n-1,abc\n3,4\n"),
    "empty_cell": dict(feats="0.5,,1\n-1,2\n3,4\n"),
    "version": dict(manifest='{"T":2,"feature_dim":2,"format_version":3,"num_nodes":3}'),
    "malformed": dict(manifest='{"T":0,"feature_dim":2,"format_version":1,"num_nodes":3}'),
    "bad_node_id": dict(d_feats="x,7,8\n"),
}


@pytest.mark.parametrize("case", sorted(MALFORMED))
def test_malformed_inputs_fail_like_reference(ref, api, tmp_path, case):
    p = _tiny(str(tmp_path), **MALFORMED[case])
    with pytest.raises(ValueError) as e_ref:
        ref.RefGraph.load_dataset(p)
    with pytest.raises((ValueError, IndexError)) as e_ours:
        _read_all(api, p)
    assert str(e_ref.value) == "invalid_argument: " + str(e_ours.value)


@pytest.mark.parametrize("edges", ["0 1\n1 2 2\n", "0\t1\n1 x 2\n2 0\n", "0 1 1 2 0", "+0 1\n1\t2\n"])
def test_edge_stream_extraction_like_reference(ref, api, tmp_path, edges):
    """`while (in >> src >> dst)`: whitespace-agnostic pairs, silent stop at the
    first failed extraction (src/dataset_io.cpp:106-110)."""
    p = _tiny(str(tmp_path), edges=edges, d_edges="", d_feats="")
    L = ref.RefGraph.load_dataset(p)
    _, (src, dst, _), _ = _read_all(api, p)
    order = np.lexsort((dst, src))
    rs, rd = L.edges(0)
    assert np.array_equal(src[order], rs) and np.array_equal(dst[order], rd)


def test_missing_file_message(api, tmp_path):
    with pytest.raises(ValueError, match="cannot open for reading: .*manifest.json"):
        api.Dataset(tmp_path / "nope")


@pytest.mark.gpu
def test_device_load_matches_reference_loader(ref, api, tmp_path):
    """load_dataset into HBM == the reference's load_dataset: CSRs and deltas
    bitwise, features = fp32 of the reference's values."""
    g = _ref_graph(ref)
    g.save_dataset(tmp_path)
    L = ref.RefGraph.load_dataset(tmp_path)
    dg = api.load_dataset(tmp_path)
    assert dg.length() == L.T
    for t in range(L.T):
        for a, b in zip(dg.in_csr(t), L.in_csr(t)):
            assert np.array_equal(a, b), t
        for a, b in zip(dg.out_csr(t), L.out_csr(t)):
            assert np.array_equal(a, b), t
        assert np.array_equal(dg.feats(t), L.feats(t).astype(np.float32)), t
        if t:
            a, b = dg.delta(t), L.delta(t)
            for k in ("del_src", "del_dst", "ins_src", "ins_dst", "changed"):
                assert np.array_equal(a[k], b[k]), (t, k)
            assert dg.change_ratio(t) == L.change_ratio(t)


@pytest.mark.gpu
def test_device_save_is_byte_identical_to_reference(ref, api, tmp_path):
    """save_dataset of the device graph writes the reference's layout: every
    file equals the reference's save of the reference's load of it, and the
    edge files equal the reference writer on the original graph."""
    g = _synth(api).to_graph()
    ours, again, theirs = tmp_path / "ours", tmp_path / "again", tmp_path / "theirs"
    api.save_dataset(g, ours)
    ref.RefGraph.load_dataset(ours).save_dataset(again)
    _ref_graph(ref).save_dataset(theirs)
    names = sorted(os.listdir(ours))
    assert names == sorted(os.listdir(again))
    for f in names:
        assert filecmp.cmp(ours / f, again / f, shallow=False), f
        if f.endswith(".edges") or f == "manifest.json":
            assert filecmp.cmp(ours / f, theirs / f, shallow=False), f


@pytest.mark.gpu
@pytest.mark.parametrize("binary", [True, False])
def test_device_round_trip(api, tmp_path, binary):
    s = _synth(api)
    g = s.to_graph()
    s.save(tmp_path / "gen", binary=binary)
    api.save_dataset(g, tmp_path / "dev", binary=binary)
    for sub in ("gen", "dev"):
        h = api.load_dataset(tmp_path / sub)
        assert h.length() == g.length()
        for t in range(g.length()):
            for a, b in zip(h.in_csr(t), g.in_csr(t)):
                assert np.array_equal(a, b), (sub, t)
            assert np.array_equal(h.feats(t), g.feats(t)), (sub, t)
            if t:
                a, b = h.delta(t), g.delta(t)
                for k in a:
                    assert np.array_equal(a[k], b[k]), (sub, t, k)
