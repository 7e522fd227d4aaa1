"""Measured FP64 FMA peak of this GPU (tr_fp64_peak: a dependent-free FMA
burst over every SM), printed as JSON."""
import ctypes as C, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1302_6945_b200 import _lib
lib = _lib.load()
p = C.c_double()
lib.tr_fp64_peak(C.byref(p))
print(json.dumps({"fp64_fma_tflops": p.value}))
