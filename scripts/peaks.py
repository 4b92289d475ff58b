import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1411_0814_b200 import rsm
print("dfma TF/s", rsm.fp64_peak_tflops(0))
print("dmma TF/s", rsm.dmma_peak_tflops(0))
