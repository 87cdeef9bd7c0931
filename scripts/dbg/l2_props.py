import torch
p = torch.cuda.get_device_properties(0)
print(p)
import ctypes
cudart = ctypes.CDLL("libcudart.so") if False else None
from cuda.bindings import runtime as rt
err, v = rt.cudaDeviceGetAttribute(rt.cudaDeviceAttr.cudaDevAttrMaxPersistingL2CacheSize, 0)
print("max persisting L2", v)
err, v = rt.cudaDeviceGetAttribute(rt.cudaDeviceAttr.cudaDevAttrL2CacheSize, 0)
print("L2", v)
err, v = rt.cudaDeviceGetAttribute(rt.cudaDeviceAttr.cudaDevAttrMaxAccessPolicyWindowSize, 0)
print("max window", v)
