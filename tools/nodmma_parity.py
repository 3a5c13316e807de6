import sys, os
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tools'); sys.path.insert(0, '/root/repo/tests')
from paper_1802_06263_b200 import _lib
_lib._lib = None
_lib.load(os.path.join(os.path.dirname(_lib._SO), "_mfb_nodmma.so"))
import parity_report, json
print(json.dumps([parity_report.report(n) for n in sys.argv[1:]], indent=1))
