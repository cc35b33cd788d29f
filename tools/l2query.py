import torch, ctypes
torch.cuda.init()
lib=ctypes.CDLL('libcudart.so') if False else None
from cuda.bindings import runtime as rt
err, v = rt.cudaDeviceGetAttribute(rt.cudaDeviceAttr.cudaDevAttrMaxPersistingL2CacheSize, 0); print("max persisting L2", v)
err, v = rt.cudaDeviceGetAttribute(rt.cudaDeviceAttr.cudaDevAttrL2CacheSize, 0); print("L2", v)
