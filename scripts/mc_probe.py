"""Does this box's GPU support NVLink SHARP multicast objects (multimem.*)?

Prints the device count and CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED per device, via the
driver API directly (no torch).  DESIGN.md §10 (why N1(i) multicast is not built)."""
import ctypes

CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED = 132

cu = ctypes.CDLL("libcuda.so.1")
assert cu.cuInit(0) == 0
n = ctypes.c_int()
cu.cuDeviceGetCount(ctypes.byref(n))
print("devices", n.value)
for d in range(n.value):
    v = ctypes.c_int()
    cu.cuDeviceGetAttribute(ctypes.byref(v), CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, d)
    print("dev", d, "multicast_supported", v.value)
