import os, sys, runpy
sys.path.insert(0, os.getcwd())
import paper_2401_11240_b200 as L
from paper_2401_11240_b200 import binding as B
orig = B.LoraPool.__init__
def init(self, *a, **k):
    orig(self, *a, **k)
    self.set_option(B.LORA_OPT_LOAD_KERNEL, int(os.environ.get("LK", "1")))
B.LoraPool.__init__ = init
sys.argv = ["bench.py", "--steps", "500", "--prefill-layers", "0", "--c4-steps", "0", "--c5-reps", "0", "--e2e-steps", "2", "--no-cpu-baseline"]
runpy.run_path("bench.py", run_name="__main__")
