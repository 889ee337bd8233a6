"""Developer timing: host-state stepping, set_state/step/get_state vs
djg_advance_host, on cfg5."""
import ctypes as C
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2106_14189_b200 import GpuDjEngine, Scenario, config_spec  # noqa: E402
from paper_2106_14189_b200 import _abi as A  # noqa: E402

sc = Scenario(config_spec("cfg5", precision=4, target=0.01, ramp_steps=100000))
eng = GpuDjEngine(sc)
lib = A.load_library()
eng.step(5)
n3 = 3 * sc.num_nodes
bufs = [torch.empty(n3, dtype=torch.float32).pin_memory() for _ in range(3)]
uc, up, st = eng.get_state()
bufs[0].numpy()[:] = uc
bufs[1].numpy()[:] = up
cur, prev, spare = (C.c_void_p(b.data_ptr()) for b in bufs)
rep = A.djg_report()
h = eng._h
for mode in ("three-call", "advance_host", "three-call", "advance_host"):
    step = C.c_int64(st)
    t0 = time.perf_counter()
    for _ in range(8):
        if mode == "three-call":
            lib.djg_set_state(h, cur, prev, step.value)
            lib.djg_step(h, 1, C.byref(rep))
            lib.djg_get_state(h, spare, None, C.byref(step))
        else:
            lib.djg_advance_host(h, cur, prev, step.value, spare, C.byref(rep))
            step.value = rep.step
        cur, prev, spare = spare, cur, prev
    print(mode, round((time.perf_counter() - t0) / 8 * 1e3, 2), "ms/step", flush=True)
    st = step.value
