import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2101_08878_b200.harness.transpose_sum import TransposeSum
n = int(sys.argv[1]); b = int(sys.argv[2])
ts = TransposeSum(n, b).setup()
ts.launch()
print("sums", list(ts.read_block_sums().items())[:3])
