import sys, time, torch
sys.path.insert(0, ".")
from paper_2102_03161_b200.configs import GEOMETRIES
from paper_2102_03161_b200.vit import VitExecutor
g = GEOMETRIES["vit-b16"]
B = 400
ex = VitExecutor(g, max_batch=B)
x = torch.randn(B, 3, 224, 224, device="cuda")
y = torch.randint(0, 1000, (B,), device="cuda")
for _ in range(3):
    ex.train_step(x, y); ex.sgd(0, 1e-3)
torch.cuda.synchronize()
for i in range(3):
    t0 = time.perf_counter(); ex.train_step(x, y); t1 = time.perf_counter(); ex.sgd(0, 1e-3); t2 = time.perf_counter()
    torch.cuda.synchronize(); t3 = time.perf_counter()
    print(f"train_step host {1e3*(t1-t0):.2f} ms, sgd host {1e3*(t2-t1):.2f}, drain {1e3*(t3-t2):.2f}")
# many steps without sync
t0 = time.perf_counter()
for i in range(5):
    ex.train_step(x, y); ex.sgd(0, 1e-3)
t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
print(f"5 steps: host {1e3*(t1-t0):.1f} ms, total {1e3*(t2-t0):.1f} ms")
