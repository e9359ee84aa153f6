import ctypes as ct
L=ct.CDLL('/root/repo/paper_1707_09598_b200/libsgiga_peaks.so')
t=ct.c_double(); m=ct.c_double()
L.sgiga_fp64_peak.argtypes=[ct.c_double,ct.POINTER(ct.c_double),ct.POINTER(ct.c_double)]
print('DFMA', L.sgiga_fp64_peak(1.0, ct.byref(t), ct.byref(m)), t.value)
L.sgiga_dmma_peak.argtypes=[ct.POINTER(ct.c_double)]
print('DMMA', L.sgiga_dmma_peak(ct.byref(t)), t.value)
