"""Host-side file-format timing: TSMESH write/read (ours vs the reference's mesh_io.hpp),
TSBMESH binary write/read, on a layered box of the given cells. args: cells (e.g. 82,123,41)."""
import os, sys, tempfile, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, 'oracle'))
import numpy as np
import paper_1710_08679_b200 as ts
from oracle import Oracle
r = Oracle("reference")
cells = tuple(int(x) for x in sys.argv[1].split(","))
ext = tuple(c * 2800.0 for c in cells)
spec = (ext, cells, (0.75 * ext[2],))
t = time.perf_counter(); m = ts.generate_box_mesh(*spec); tg = time.perf_counter() - t
a = r.box_mesh(*spec, 1)
d = tempfile.mkdtemp(dir="/tmp")
p1, p2, p3 = os.path.join(d, "a.tsmesh"), os.path.join(d, "b.tsmesh"), os.path.join(d, "c.tsbmesh")
def tm(f, *a):
    t = time.perf_counter(); out = f(*a); return time.perf_counter() - t, out
w_ours, _ = tm(ts.write_mesh, m, p1)
w_ref, _ = tm(r.write_mesh, a, p2)
same = open(p1, 'rb').read() == open(p2, 'rb').read()
r_ours, m2 = tm(ts.read_mesh, p1)
r_ref, _ = tm(r.read_mesh, p1)
wb, _ = tm(ts.write_mesh_binary, m, p3)
rb, _ = tm(ts.read_mesh_binary, p3)
print(dict(nodes=m.node_count(), elems=m.element_count(), bytes=os.path.getsize(p1), bin_bytes=os.path.getsize(p3), generate_s=round(tg,3),
           write_ours=round(w_ours,3), write_ref=round(w_ref,3), identical=same, read_ours=round(r_ours,3), read_ref=round(r_ref,3),
           write_bin=round(wb,3), read_bin=round(rb,3), threads=os.cpu_count()))
import shutil; shutil.rmtree(d)
