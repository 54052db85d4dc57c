"""File formats either side of the solve against the
reference's own readers/writers (mesh_io.hpp, solution_io.hpp, compiled from
the reference headers into oracle/_ref): byte-identical files, identical
arrays after reading either side's files, and the same ParseError /
ValidationError (class, line, message) on malformed input. Re-states
test_mesh.cpp:120-188 (round trip, truncation, negative volume, garbage
header) and test_cli.cpp's TSVEC checks. Host-only code: runs without a GPU,
except the device-streamed TSVEC path (marked gpu)."""
import os

import numpy as np
import pytest

import paper_1710_08679_b200 as ts

SPECS = [
    ((1723.0, 911.0, 400.5), (2, 3, 2), (133.7,), 1),  # test_mesh.cpp:121-125
    ((8000.0, 8000.0, 6000.0), (5, 4, 3), (1234.5678, 4500.0), 2),
    ((1.0, 1.0, 1.0), (1, 1, 1), (), 0),
    ((3.0e7, 1.0e-3, 7.77), (3, 2, 2), (), 1),
]


def product_mesh(a):
    return ts.Mesh.from_arrays(a.coords, a.tets10, a.material_id, a.vertex_count, a.bc_node, a.bc_axis)


def same_arrays(m: ts.Mesh, a, with_bc=True):
    arr = m.arrays()
    assert m.vertex_count == a.vertex_count
    assert np.array_equal(arr["coords"].view(np.uint64), np.ascontiguousarray(a.coords).view(np.uint64))
    assert np.array_equal(arr["tets10"], a.tets10)
    assert np.array_equal(arr["material_id"], a.material_id)
    if with_bc:
        assert np.array_equal(arr["bc_node"], a.bc_node)
        assert np.array_equal(arr["bc_axis"], a.bc_axis)


def read_bytes(p):
    with open(p, "rb") as f:
        return f.read()


@pytest.mark.parametrize("spec", SPECS)
def test_tsmesh_bytes_and_round_trip(reference, tmp_path, spec):
    a = reference.box_mesh(*spec)
    m = product_mesh(a)
    ours, theirs = tmp_path / "ours.tsmesh", tmp_path / "ref.tsmesh"
    ts.write_mesh(m, ours)
    reference.write_mesh(a, theirs)
    assert read_bytes(ours) == read_bytes(theirs)
    # each side reads the other's file into identical arrays (no Dirichlet list in TSMESH)
    same_arrays(ts.read_mesh(theirs), a, with_bc=False)
    r = reference.read_mesh(ours)
    assert np.array_equal(r.coords.view(np.uint64), a.coords.view(np.uint64))
    assert np.array_equal(r.tets10, a.tets10) and np.array_equal(r.material_id, a.material_id)
    # Dirichlet sidecar
    ts.write_dirichlet(m, tmp_path / "ours.dirichlet")
    reference.write_dirichlet(a, tmp_path / "ref.dirichlet")
    assert read_bytes(tmp_path / "ours.dirichlet") == read_bytes(tmp_path / "ref.dirichlet")
    back = ts.read_mesh(ours)
    ts.read_dirichlet(back, tmp_path / "ref.dirichlet")
    same_arrays(back, a)
    assert np.array_equal(back.dirichlet_mask(), a.dirichlet_mask())
    assert not [p for p in os.listdir(tmp_path) if ".tmp" in p]  # atomic_write leaves no temporaries


def test_generated_mesh_writes_like_reference(reference, tmp_path):
    spec = ((1723.0, 911.0, 400.5), (4, 3, 2), (133.7,), 1)
    ts.write_mesh(ts.generate_box_mesh(*spec[:3]), tmp_path / "a.tsmesh")
    reference.write_mesh(reference.box_mesh(*spec), tmp_path / "b.tsmesh")
    assert read_bytes(tmp_path / "a.tsmesh") == read_bytes(tmp_path / "b.tsmesh")


def both_fail_alike(reference, path):
    """The product and the reference reject `path` with the same class and message."""
    with pytest.raises(ts.ValidationError) as ours:
        ts.read_mesh(path)
    with pytest.raises(Exception) as theirs:
        reference.read_mesh(path)
    assert str(ours.value) == str(theirs.value)
    assert isinstance(ours.value, ts.ParseError) == (theirs.value.code == 7)
    return str(ours.value)


def unit_mesh_text(reference, tmp_path):
    a = reference.box_mesh((1.0, 1.0, 1.0), (1, 1, 1), (), 0)
    p = tmp_path / "u.tsmesh"
    reference.write_mesh(a, p)
    return a, p, read_bytes(p).decode().splitlines(keepends=True)


def test_truncated_file_reports_position(reference, tmp_path):  # test_mesh.cpp:146-163
    a, p, lines = unit_mesh_text(reference, tmp_path)
    for keep in (0, 1, 2, 10, len(lines) - 1):
        p.write_text("".join(lines[:keep]))
        msg = both_fail_alike(reference, p)
        assert f":{keep + 1}: unexpected end of file" in msg


def test_negative_volume_named(reference, tmp_path):  # test_mesh.cpp:165-178
    a = reference.box_mesh((1.0, 1.0, 1.0), (1, 1, 1), (), 0)
    a.tets10[3, [0, 1]] = a.tets10[3, [1, 0]]
    p = tmp_path / "neg.tsmesh"
    reference.write_mesh(a, p)
    msg = both_fail_alike(reference, p)
    assert "element 3" in msg and "non-positive volume" in msg


def test_garbage_header(reference, tmp_path):  # test_mesh.cpp:180-188
    p = tmp_path / "bad.tsmesh"
    for text in ("NOTAMESH 9\n", "TSMESH 2\n", "TSMESH\n", "", "TSMESH 1\nnodes 3 vertex_nodes 2\n",
                 "TSMESH 1\nnodes -1 vertex_nodes 0 tets 0\n", "TSMESH 1\nnode 0 vertex_nodes 0 tets 0\n"):
        p.write_text(text)
        both_fail_alike(reference, p)


def test_empty_mesh_and_line_endings(reference, tmp_path):
    p = tmp_path / "e.tsmesh"
    p.write_text("TSMESH 1\nnodes 0 vertex_nodes 0 tets 0")  # no trailing newline
    assert ts.read_mesh(p).node_count() == 0 and reference.read_mesh(p).n_nodes == 0
    a, q, lines = unit_mesh_text(reference, tmp_path)
    q.write_bytes("".join(ln.replace("\n", "\r\n") for ln in lines).encode())  # CRLF
    same_arrays(ts.read_mesh(q), a, with_bc=False)
    q.write_bytes(("".join(lines) + "trailing garbage is ignored\n").encode())
    same_arrays(ts.read_mesh(q), a, with_bc=False)
    reference.read_mesh(q)


# numeric tokens as istream >> double reads them (num_get + strtod)
COORD_TOKENS = ["1e5", "+3", ".5", "1.", "-0", "1e", "1e+", "0x10", "inf", "nan", "1e999", "-1e999", "1e-400",
                "4.9e-324", "00012", "1.5e+3x", "--1", "+-1", ".", "-.5e-2", "1,5", "٣", "1e5.5", " \t 2 "]
INT_TOKENS = ["+5", "-0", "5.0", "0x3", "99999999999", "2147483647", "-2147483649", "5e1", "+", "07"]


@pytest.mark.parametrize("tok", COORD_TOKENS)
def test_coordinate_tokens_parse_like_reference(reference, tmp_path, tok):
    a, p, lines = unit_mesh_text(reference, tmp_path)
    # an extra node no element references: only the parse decides (validate_mesh ignores it)
    n = a.n_nodes
    lines[1] = lines[1].replace(f"nodes {n} ", f"nodes {n + 1} ")
    lines.insert(2 + n, f"0.25 {tok} 7\n")
    p.write_bytes("".join(lines).encode())
    try:
        r = reference.read_mesh(p)
    except Exception as e:
        with pytest.raises(ts.ValidationError) as ours:
            ts.read_mesh(p)
        assert str(ours.value) == str(e)
        return
    m = ts.read_mesh(p)
    assert np.array_equal(m.coords.view(np.uint64), r.coords.view(np.uint64)) and m.node_count() == n + 1


@pytest.mark.parametrize("tok", INT_TOKENS)
@pytest.mark.parametrize("slot", [0, 4, 10])
def test_element_tokens_parse_like_reference(reference, tmp_path, tok, slot):
    a, p, lines = unit_mesh_text(reference, tmp_path)
    n = a.n_nodes
    words = lines[2 + n].split()
    words[slot] = tok
    lines[2 + n] = " ".join(words) + "\n"
    p.write_bytes("".join(lines).encode())
    try:
        r = reference.read_mesh(p)
    except Exception as e:
        with pytest.raises(ts.ValidationError) as ours:
            ts.read_mesh(p)
        assert str(ours.value) == str(e)
        return
    m = ts.read_mesh(p)
    assert np.array_equal(m.tets10, r.tets10) and np.array_equal(m.material_id, r.material_id)


def test_validation_errors_match(reference, tmp_path):
    a = reference.box_mesh((2.0, 1.0, 1.0), (2, 1, 1), (), 0)
    cases = []
    b = reference.box_mesh((2.0, 1.0, 1.0), (2, 1, 1), (), 0)
    b.tets10[5, 7] = b.n_nodes + 3  # out of range node
    cases.append(b)
    b = reference.box_mesh((2.0, 1.0, 1.0), (2, 1, 1), (), 0)
    b.coords[b.tets10[4, 6]] += 1e-3  # displaced edge node
    cases.append(b)
    b = reference.box_mesh((2.0, 1.0, 1.0), (2, 1, 1), (), 0)
    b.tets10[8, 2] = -1
    cases.append(b)
    for k, b in enumerate(cases):
        p = tmp_path / f"v{k}.tsmesh"
        with open(p, "w") as f:
            f.write(f"TSMESH 1\nnodes {b.n_nodes} vertex_nodes {b.vertex_count} tets {b.n_elems}\n")
            for c in b.coords:
                f.write("%.17g %.17g %.17g\n" % tuple(c))
            for t, mid in zip(b.tets10, b.material_id):
                f.write(" ".join(str(x) for x in t) + f" {mid}\n")
        msg = both_fail_alike(reference, p)
        assert "mesh:" in msg
    p = tmp_path / "vc.tsmesh"
    p.write_text("TSMESH 1\nnodes 0 vertex_nodes 4 tets 0\n")
    both_fail_alike(reference, p)
    del a


def test_dirichlet_errors_match(reference, tmp_path):
    a = reference.box_mesh((1.0, 1.0, 1.0), (1, 1, 1), (), 1)
    m = product_mesh(a)
    p = tmp_path / "d.dirichlet"
    for text in ("0 0\n\n3 2\n", "0 3\n", "0\n", "-1 0\n", f"{a.n_nodes} 1\n", "1 1\n \n", "", "2 1"):
        p.write_text(text)
        try:
            r = reference.read_dirichlet(a, p)
        except Exception as e:
            with pytest.raises(ts.ParseError) as ours:
                ts.read_dirichlet(m, p)
            assert str(ours.value) == str(e)
            continue
        ts.read_dirichlet(m, p)
        same_arrays(m, r)


def test_tsvec_bytes_and_round_trip(reference, tmp_path):
    rng = np.random.default_rng(3)
    for n, b in ((5, 1), (17, 4), (0, 3), (40, 16)):
        u = rng.standard_normal((3 * n, b))
        ts.write_solution(u, tmp_path / "a.tsvec")
        reference.write_solution(tmp_path / "b.tsvec", u)
        assert read_bytes(tmp_path / "a.tsvec") == read_bytes(tmp_path / "b.tsvec")
        got = ts.read_solution(tmp_path / "b.tsvec")
        assert got.shape == (3 * n, b) and np.array_equal(got.view(np.uint64), u.view(np.uint64))
        assert np.array_equal(reference.read_solution(tmp_path / "a.tsvec"), u)


def test_tsvec_errors_match(reference, tmp_path):
    u = np.arange(3 * 4 * 2, dtype=np.float64).reshape(12, 2)
    reference.write_solution(tmp_path / "g.tsvec", u)
    good = read_bytes(tmp_path / "g.tsvec")
    head, payload = good.split(b"DATA\n", 1)
    p = tmp_path / "x.tsvec"
    variants = [
        head + b"DATA\n" + payload[:-1],                      # truncated payload
        head.replace(b"TSVEC 1", b"TSVEC 2") + b"DATA\n" + payload,
        head.replace(b"axes 3", b"axes 2") + b"DATA\n" + payload,
        head.replace(b"float64", b"float32") + b"DATA\n" + payload,
        head.replace(b"little", b"big") + b"DATA\n" + payload,
        head.replace(b"node_axis_batch", b"batch_node_axis") + b"DATA\n" + payload,
        head.replace(b"batch 2", b"batch 0") + b"DATA\n" + payload,
        head.replace(b"nodes 4", b"nodes x") + b"DATA\n" + payload,
        head.replace(b"batch 2\n", b"") + b"DATA\n" + payload,
        b"TSVEC 1\nnodes 4\n",
        b"",
        good + b"extra bytes are ignored",
    ]
    for v in variants:
        p.write_bytes(v)
        try:
            r = reference.read_solution(p)
        except Exception as e:
            with pytest.raises(ts.ParseError) as ours:
                ts.read_solution(p)
            assert str(ours.value) == str(e)
            continue
        assert np.array_equal(ts.read_solution(p), r)


@pytest.mark.parametrize("spec", SPECS[:2])
def test_binary_mesh_round_trip(reference, tmp_path, spec):
    a = reference.box_mesh(*spec)
    m = product_mesh(a)
    p = tmp_path / "m.tsbmesh"
    ts.write_mesh_binary(m, p)
    same_arrays(ts.read_mesh_binary(p), a)
    raw = read_bytes(p)
    p.write_bytes(raw[:-3])
    with pytest.raises(ts.ParseError, match="truncated binary payload"):
        ts.read_mesh_binary(p)
    p.write_bytes(raw.replace(b"TSBMESH 1", b"TSBMESH 3", 1))
    with pytest.raises(ts.ParseError, match="unsupported version"):
        ts.read_mesh_binary(p)
    b = reference.box_mesh(*spec)
    b.tets10[2, [0, 1]] = b.tets10[2, [1, 0]]
    ts.write_mesh_binary(product_mesh(b), p)
    with pytest.raises(ts.ValidationError, match="element 2 has non-positive volume"):
        ts.read_mesh_binary(p)


def test_missing_files(tmp_path):
    for fn in (ts.read_mesh, ts.read_mesh_binary, ts.read_solution):
        with pytest.raises(ts.ValidationError, match="cannot open"):
            fn(tmp_path / "nope")
    with pytest.raises(ts.ValidationError, match="cannot open for writing"):
        ts.write_solution(np.zeros((3, 1)), tmp_path / "no_dir" / "x.tsvec")


@pytest.mark.gpu
def test_tsvec_device_streaming(tmp_path):
    import torch
    # > 2 staging chunks (64 MB each) so the double-buffered pipeline wraps around
    u = torch.randn(3 * 1_500_000, 6, dtype=torch.float64, device="cuda")
    p = tmp_path / "d.tsvec"
    ts.write_solution(u, p)
    host = u.cpu().numpy()
    ts.write_solution(host, tmp_path / "h.tsvec")
    assert read_bytes(p) == read_bytes(tmp_path / "h.tsvec")
    back = ts.read_solution(p, device="cuda")
    assert torch.equal(back, u)


def test_unstructured_mesh_files(reference, tmp_path):
    """Non-round coordinates (jittered vertices), scrambled numbering: %.17g text, the
    binary mesh and TSVEC stay byte-identical / bit-exact against the reference."""
    from test_unstructured_gpu import scrambled_mesh
    a, m = scrambled_mesh(reference, (3000.0, 2000.0, 1500.0), (5, 4, 3), 21)
    ts.write_mesh(m, tmp_path / "u.tsmesh")
    reference.write_mesh(a, tmp_path / "r.tsmesh")
    assert read_bytes(tmp_path / "u.tsmesh") == read_bytes(tmp_path / "r.tsmesh")
    ts.write_dirichlet(m, tmp_path / "u.dirichlet")
    reference.write_dirichlet(a, tmp_path / "r.dirichlet")
    assert read_bytes(tmp_path / "u.dirichlet") == read_bytes(tmp_path / "r.dirichlet")
    back = ts.read_mesh(tmp_path / "r.tsmesh")
    ts.read_dirichlet(back, tmp_path / "r.dirichlet")
    same_arrays(back, a)
    ts.write_mesh_binary(back, tmp_path / "u.tsbmesh")
    same_arrays(ts.read_mesh_binary(tmp_path / "u.tsbmesh"), a)


# ---------------------------------------------------------------- Green's-sweep files
from paper_1710_08679_b200 import greens as G  # noqa: E402


def same_bank(a, b):
    for k in ("values", "obs_points", "centers", "radii"):
        assert np.array_equal(np.asarray(a[k]).view(np.uint64), np.asarray(b[k]).view(np.uint64)), k
    for k in ("obs_axes", "directions"):
        assert np.array_equal(a[k], b[k]), k


def test_fault_faces_files(reference, tmp_path):
    rng = np.random.default_rng(4)
    faces = rng.integers(0, 10**6, (37, 3)).astype(np.int32)
    G.write_fault_faces(faces, tmp_path / "a.tsfault")
    reference.write_fault_faces(tmp_path / "b.tsfault", faces)
    assert read_bytes(tmp_path / "a.tsfault") == read_bytes(tmp_path / "b.tsfault")
    assert np.array_equal(G.read_fault_faces(tmp_path / "b.tsfault"), faces)
    p = tmp_path / "x.tsfault"
    good = read_bytes(tmp_path / "a.tsfault").decode().splitlines(keepends=True)
    for text in ("", "TSFAULT 2\nfaces 1\n1 2 3\n", "TSFAULT 1\nfaces 0\n", "TSFAULT 1\nfaces 2\n1 2 3\n",
                 "TSFAULT 1\nfaces 1\n1 2\n", "TSFAULT 1\nfacez 1\n1 2 3\n", "".join(good[:5]),
                 "TSFAULT 1\nfaces 1\n1 2 3 4 extra\n"):
        p.write_text(text)
        try:
            want = reference.read_fault_faces(p)
        except Exception as e:
            with pytest.raises(ts.ValidationError) as ours:
                G.read_fault_faces(p)
            assert str(ours.value) == str(e)
            continue
        assert np.array_equal(G.read_fault_faces(p), want)


def test_observations_file(reference, tmp_path):
    p = tmp_path / "obs.txt"
    cases = [
        "# surface stations\n1000 2000 6000 x\n3000.5 4000 6000 y  # trailing\n\n5e3 4e3 6e3 2\n",
        "abc\n1 2 3 0\n",                  # non-numeric line skipped
        "1 2 3 w\n",                      # bad axis
        "1 2\n",                          # short line
        "# nothing\n\n",                  # empty -> ValidationError
        "1 2 3 z\n4 5 6 1",               # no final newline
    ]
    for text in cases:
        p.write_text(text)
        try:
            want = reference.read_observations(p)
        except Exception as e:
            with pytest.raises(ts.ValidationError) as ours:
                G.read_observations(p)
            assert str(ours.value) == str(e)
            continue
        got = G.read_observations(p)
        assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1])


def test_greens_bank_files(reference, tmp_path):
    rng = np.random.default_rng(8)
    R, K = 7, 5
    bank = rng.standard_normal((R, K)) * 1e-3
    pts = rng.uniform(0, 8000, (R, 3))
    axes = rng.integers(0, 3, R).astype(np.int32)
    centers = rng.uniform(0, 8000, (K, 3))
    dirs = rng.integers(0, 2, K).astype(np.int32)
    radii = rng.uniform(500, 2000, K)
    G.write_greens_bank(tmp_path / "a.tsgreens", bank, pts, axes, centers, dirs, radii)
    reference.write_greens_bank(tmp_path / "b.tsgreens", bank, pts, axes, centers, dirs, radii)
    assert read_bytes(tmp_path / "a.tsgreens") == read_bytes(tmp_path / "b.tsgreens")
    same_bank(G.read_greens_bank(tmp_path / "b.tsgreens"), reference.read_greens_bank(tmp_path / "a.tsgreens"))
    good = read_bytes(tmp_path / "a.tsgreens")
    head, payload = good.split(b"DATA\n", 1)
    p = tmp_path / "x.tsgreens"
    for v in (head + b"DATA\n" + payload[:-8], head.replace(b"TSGREENS 1", b"TSGREENS 0") + b"DATA\n" + payload,
              head.replace(b"rows 7", b"rows 0") + b"DATA\n" + payload, head.replace(b" dip ", b" dup ", 1)
              + b"DATA\n" + payload, head.replace(b"obs ", b"ob ", 1) + b"DATA\n" + payload, head, b""):
        p.write_bytes(v)
        try:
            want = reference.read_greens_bank(p)
        except Exception as e:
            with pytest.raises(ts.ValidationError) as ours:
                G.read_greens_bank(p)
            assert str(ours.value) == str(e)
            continue
        same_bank(G.read_greens_bank(p), want)
