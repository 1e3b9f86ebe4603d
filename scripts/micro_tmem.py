import sys; sys.path.insert(0,'/root/repo')
from paper_2411_10958_b200 import sage2
for w in (0,1,10,11):
    print(w, sage2.MICRO[w], round(sage2.microbench(w, 4096),1))
