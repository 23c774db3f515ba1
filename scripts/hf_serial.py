import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2509_20563_b200 as fz
from paper_2509_20563_b200 import data
from paper_2509_20563_b200.core import ErrorBoundSpec, ErrorMode, Field
lib = ctypes.CDLL(os.environ["FZB_SO"])
for dims, pipe in (((100, 500, 500), "default"), ((1800, 3600), "quality")):
    x = data.smooth_trig_host(dims, 0)
    a = fz.compress(Field(dims, x), ErrorBoundSpec(ErrorMode.VALUE_RANGE_RELATIVE, 1e-4), pipe)
    v = ctypes.c_uint32(0)
    lib.fzb_debug_hf_serial(ctypes.byref(v))
    print(dims, pipe, "serial merge levels so far:", v.value)
