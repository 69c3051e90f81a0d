"""Probe: does this box support NVLink multicast objects (NVLS)?"""
import ctypes
cu = ctypes.CDLL("libcuda.so.1")
assert cu.cuInit(0) == 0
n = ctypes.c_int()
cu.cuDeviceGetCount(ctypes.byref(n))
for d in range(n.value):
    dev = ctypes.c_int()
    cu.cuDeviceGet(ctypes.byref(dev), d)
    for name, attr in (("MULTICAST_SUPPORTED", 132), ("HANDLE_TYPE_FABRIC_SUPPORTED", 128),
                       ("HANDLE_TYPE_POSIX_FD_SUPPORTED", 101), ("VIRTUAL_MEMORY_MANAGEMENT_SUPPORTED", 102)):
        v = ctypes.c_int(-1)
        rc = cu.cuDeviceGetAttribute(ctypes.byref(v), attr, dev)
        print(d, name, v.value, "rc", rc)
