"""Developer timeline of one djg_advance_host call on cfg5 (pinned host
buffers): run with DJG_TRACE_HOST=1; the engine prints event times (ms from
the call's start) per stream to stderr."""
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
eng.step(3)
n3 = 3 * sc.num_nodes
bufs = [torch.empty(n3, dtype=torch.float32).pin_memory() for _ in range(3)]
uc, up, st = eng.get_state()
bufs[0].numpy()[:] = uc
bufs[1].numpy()[:] = up
cur, prev, spare = (C.c_void_p(b.data_ptr()) for b in bufs)
rep = A.djg_report()
for i in range(3):
    t0 = time.perf_counter()
    rc = lib.djg_advance_host(eng._h, cur, prev, st, spare, C.byref(rep))
    print(f"call {i}: rc {rc} {lib.djg_last_error(eng._h).decode() if rc else ''} "
          f"{1e3 * (time.perf_counter() - t0):.3f} ms wall", file=sys.stderr, flush=True)
    st = rep.step
    cur, prev, spare = spare, cur, prev
