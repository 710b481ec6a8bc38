"""Per-phase decode trace (scripts/trace_decode.py) on pools loaded by LORA_OPT_LOAD_KERNEL=LK
(env), to see which phase differs in the occasional slow mode.  usage: LK=1 python this.py"""
import os
import runpy
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2401_11240_b200 import binding as B  # noqa: E402

orig = B.LoraPool.__init__


def init(self, *a, **k):
    orig(self, *a, **k)
    self.set_option(B.LORA_OPT_LOAD_KERNEL, int(os.environ.get("LK", "1")))


B.LoraPool.__init__ = init
sys.argv = ["trace_decode.py", "c2", "32"]
runpy.run_path(os.path.join(os.path.dirname(os.path.abspath(__file__)), "trace_decode.py"), run_name="__main__")
