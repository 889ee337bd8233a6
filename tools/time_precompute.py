"""Developer timing: djg_create_from_mesh (DjEngine construction: records,
adjacency, slot layout) with the precompute on the host vs on the device,
plus the device lump_mass / characteristic length, on a SURVEY config."""
import ctypes as C
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2106_14189_b200 import Scenario, config_spec  # noqa: E402
from paper_2106_14189_b200 import _abi as A  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
sc = Scenario(config_spec(name, precision=4))
img = sc.image()
lib = A.load_library()
for flags, tag in ((0, "host"), (A.DJG_FLAG_DEVICE_PRECOMPUTE, "device")):
    m = A.djg_mesh_desc()
    m.precision, m.kind = 4, sc.spec.c.kind
    m.num_nodes, m.num_elements = sc.num_nodes, sc.num_elements
    m.nodes = img["nodes"].ctypes.data_as(C.c_void_p)
    m.conn = img["conn"].ctypes.data_as(C.c_void_p)
    m.material = sc.spec.c.material
    m.c_hg, m.flags, m.threads = 0.1, flags, 0
    h = C.c_void_p()
    t0 = time.perf_counter()
    rc = lib.djg_create_from_mesh(C.byref(m), C.byref(h))
    t1 = time.perf_counter()
    out = dict(cfg=name, precompute=tag, rc=rc, create_s=round(t1 - t0, 3))
    if flags:
        import numpy as np
        mass = np.zeros(sc.num_nodes, np.float32)
        lib.djg_lump_mass(h, mass.ctypes.data_as(C.c_void_p))
        out["mass_equal_host_builder"] = bool(np.array_equal(mass, img["mass"]))
    lib.djg_destroy(h)
    print(json.dumps(out), flush=True)
