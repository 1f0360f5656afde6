cd $GRAFT_REPO_ROOT
PASE_LIB=paper_2407_04001_b200/libpase_btdbg.so timeout 300 python -c "
from paper_2407_04001_b200 import pase, zoo
for w in ['transformer','gnmt','inception_v3']:
    g,p=zoo.bench_graph(w)
    c=pase.Context(g,p,device=0)
    for i in range(3): c.solve()
    print(w, c.stats()['ms_solve'], flush=True)
" 2>&1 | tail -60
