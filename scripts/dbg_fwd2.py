import sys, os; sys.path.insert(0, os.getcwd())
import numpy as np
from paper_1810_13100_b200 import ncsg, _build
if len(sys.argv) > 1: _build.LIB = os.path.abspath(sys.argv[1])
R = ncsg.RadonMap(16, 12, 25)
print(sys.argv[1:], "sum", R.forward(np.ones((16,16))).sum())
