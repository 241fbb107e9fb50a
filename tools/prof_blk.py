import ctypes, os, subprocess, sys
sys.argv = ["diag.py", "--reps", "1"]
sys.path.insert(0, os.getcwd())
import tools.diag as dg
dg.main()
from paper_1708_06290_b200 import _lib
L = _lib.load()
arr = (ctypes.c_ulonglong * 4)()
L.ss_blk_prof(arr)
tot = sum(arr[:3])
print("chain %.1f%%  reverse %.1f%%  passes %.1f%%  (total %.3e warp-cycles)" % (100*arr[0]/tot, 100*arr[1]/tot, 100*arr[2]/tot, tot))
