"""Print the GPU box's host facts and the SHA-256 of a generated config field
(to check that numpy on the box reproduces this container's fields)."""
import hashlib, os, subprocess, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from paper_2007_09625_b200 import synthetic
print("nproc", os.cpu_count())
print(subprocess.run(["free", "-g"], capture_output=True, text=True).stdout)
print([l for l in subprocess.run(["lscpu"], capture_output=True, text=True).stdout.splitlines() if "Model name" in l or "Socket" in l or "NUMA node(s)" in l])
for dims in ((100, 500, 500), (1800, 3600)):
    t = time.time()
    f = synthetic.generate_field("smooth", dims, seed=1).astype(np.float32)
    print(dims, hashlib.sha256(f.tobytes()).hexdigest(), f"{time.time()-t:.1f}s")
f = synthetic.generate_field("sparse-near-zero", (128, 128, 128), seed=1).astype(np.float32)
print("sparse128", hashlib.sha256(f.tobytes()).hexdigest())
