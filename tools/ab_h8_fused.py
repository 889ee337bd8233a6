import json, sys, torch
sys.path.insert(0, ".")
from paper_2106_14189_b200 import GpuDjEngine, Scenario, box_spec, _abi as A
d = int(sys.argv[1]); model = sys.argv[2]
sc = Scenario(box_spec(kind="H8", model=model, divisions=d, precision=4, target=0.01, ramp_steps=100000))
for fl in (A.DJG_FLAG_FUSED, A.DJG_FLAG_NO_FUSED):
    with GpuDjEngine(sc, flags=fl) as eng:
        eng.step(10)
        s = torch.cuda.ExternalStream(eng.stream)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); a.record(s); eng.step_async(100); b.record(s); b.synchronize()
        print(json.dumps(dict(d=d, model=model, fused=eng.info()["fused"], us=round(a.elapsed_time(b) / 100 * 1e3, 1))))
