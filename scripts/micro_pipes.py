import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_10958_b200 import sage2
for w in (2, 3, 7, 8, 9):
    print(w, sage2.MICRO[w], sage2.microbench(w, 2048))
