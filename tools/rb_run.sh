cd $GRAFT_REPO_ROOT
python tools/rb_probe.py qft cfg4 2>&1 | grep RB
RB=3 LQ_JIT_MINBLOCKS=2 python tools/rb_probe.py qft cfg4 2>&1 | grep RB
RB=3 LQ_JIT_MINBLOCKS=3 python tools/rb_probe.py qft cfg4 2>&1 | grep RB
RB=4 LQ_JIT_MINBLOCKS=4 python tools/rb_probe.py qft 2>&1 | grep RB
