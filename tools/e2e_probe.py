"""Is the e2e (Trainer.step_async) path host- or device-bound? Times K async steps
(a) as bench.py does and (b) with a queued GPU spin in front so the host enqueues every
step before the device reaches them (device time only), plus host enqueue time per step."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from bench import he_init, synthetic_batch  # noqa: E402
from paper_1811_01532_b200 import models, planner, trainer  # noqa: E402

model = sys.argv[1] if len(sys.argv) > 1 else "alexnet"
b = 128 if model == "alexnet" else 32
K = 10
g = models.MODELS[model](b)
tp = trainer.plan_training(g, 1, planner.load_profile("b200"), force_d=1)
tr = trainer.Trainer(tp, precision=3, use_graph=True, variables=he_init(g))
batch = synthetic_batch(g, 0, b)
tr.load(batch)
for _ in range(5):
    tr.run()
for _ in range(3):
    tr.step_async(batch)
torch.cuda.synchronize()
st = torch.cuda.current_stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
for _ in range(K):
    tr.run()
e1.record(st)
torch.cuda.synchronize()
print(f"device-resident run(): {e0.elapsed_time(e1) / K:.3f} ms/step")
for spin in (False, True):
    torch.cuda.synchronize()
    if spin:
        torch.cuda._sleep(200_000_000)
    e0.record(st)
    tr.copy_stream.wait_stream(st)
    h0 = time.perf_counter()
    for _ in range(K):
        tr.step_async(batch)
    h1 = time.perf_counter()
    e1.record(st)
    tr.last_loss()
    torch.cuda.synchronize()
    print(f"step_async spin={spin}: device {e0.elapsed_time(e1) / K:.3f} ms/step, host enqueue "
          f"{(h1 - h0) * 1e3 / K:.3f} ms/step")
# (c) device-resident steps while an unrelated pinned H2D stream runs alongside
n = 128 * 224 * 224 * 3
h = torch.empty(n, dtype=torch.float32).pin_memory()
d = torch.empty(n, dtype=torch.float32, device="cuda")
cs = torch.cuda.Stream()
torch.cuda.synchronize()
with torch.cuda.stream(cs):
    for _ in range(40):
        d.copy_(h, non_blocking=True)
e0.record(st)
for _ in range(K):
    tr.run()
e1.record(st)
torch.cuda.synchronize()
print(f"run() beside a concurrent H2D stream: {e0.elapsed_time(e1) / K:.3f} ms/step")
# (d) the input path alone: bind_overlapped (H2D on the copy stream + pack on compute)
torch.cuda.synchronize()
e0.record(st)
tr.copy_stream.wait_stream(st)
for _ in range(K):
    tr.prog.bind_overlapped(batch, tr.copy_stream)
e1.record(st)
torch.cuda.synchronize()
print(f"bind_overlapped alone: {e0.elapsed_time(e1) / K:.3f} ms/step (H2D-bound when serialised)")
torch.cuda._sleep(100_000_000)
cs.wait_stream(st)
e0.record(st)
for _ in range(K):
    tr.prog.bind_overlapped(batch, tr.copy_stream)
    tr.run()
e1.record(st)
torch.cuda.synchronize()
print(f"bind_overlapped + run, spin: {e0.elapsed_time(e1) / K:.3f} ms/step")
# (e) step_async with the labels only (images stay resident): the H2D volume's share
lab = {"labels": batch["labels"]}
tr2 = trainer.Trainer(tp, precision=3, use_graph=True, variables=he_init(g))
tr2.load(batch)
for _ in range(3):
    tr2.step_async(lab)
torch.cuda.synchronize()
for spin in (False, True):
    if spin:
        torch.cuda._sleep(200_000_000)
    e0.record(st)
    tr2.copy_stream.wait_stream(st)
    for _ in range(K):
        tr2.step_async(lab)
    e1.record(st)
    torch.cuda.synchronize()
    print(f"step_async labels only spin={spin}: {e0.elapsed_time(e1) / K:.3f} ms/step")
# (f) the staging -> layout pack alone (device time)
from paper_1811_01532_b200 import _native as N  # noqa: E402
stg = tr.prog.staging(batch, 0)
torch.cuda.synchronize()
e0.record(st)
for _ in range(K):
    tr.prog.pack_staged(stg, N.stream_ptr())
e1.record(st)
torch.cuda.synchronize()
print(f"pack_staged alone: {e0.elapsed_time(e1) / K:.4f} ms/step")
