"""Print the device's L2 size, persisting-L2 maximum and access-policy window maximum (GPU box)."""
import json

import torch
from cuda.bindings import runtime as rt

dev = torch.cuda.current_device()
out = {}
for name in ("cudaDevAttrL2CacheSize", "cudaDevAttrMaxPersistingL2CacheSize", "cudaDevAttrMaxAccessPolicyWindowSize"):
    err, v = rt.cudaDeviceGetAttribute(getattr(rt.cudaDeviceAttr, name), dev)
    out[name] = v
print(json.dumps(out))
