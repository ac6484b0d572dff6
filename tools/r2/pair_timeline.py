import sys
sys.argv = ["x", "gemm8192", "16"]
sys.path.insert(0, ".")
import paper_1705_09864_b200 as bnn
from paper_1705_09864_b200 import _lib
bnn.load_library()
_lib.call("bnn_debug_set", _lib.DEBUG_PAIR_KW32, 1)
exec(open("tools/umma_stages_conv.py").read())
