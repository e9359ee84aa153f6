"""compare two dump_sys.py outputs bitwise"""
import sys
import numpy as np
a, b = np.load(sys.argv[1]), np.load(sys.argv[2])
for k in a.files:
    same = np.array_equal(a[k], b[k])
    print(k, "bitwise" if same else "DIFF max %.2e" % np.abs(a[k] - b[k]).max())
