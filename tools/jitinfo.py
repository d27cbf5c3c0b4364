import ctypes as C, sys
sys.path.insert(0, '/root/repo')
def info(tag):
    from paper_2507_13204_b200 import _cabi
    a,b,c=C.c_int(),C.c_int(),C.c_int()
    _cabi.check(_cabi.lib().krn_jit_info(C.byref(a),C.byref(b),C.byref(c)))
    print(tag, a.value,b.value,c.value, [l.split()[-1] for l in open('/proc/self/maps') if 'nvrtc' in l and 'r-xp' in l])
if sys.argv[1]=='torchfirst':
    import torch
    x=torch.rand(1000,device='cuda',dtype=torch.float64)*2-1
    y=torch.from_numpy(__import__('numpy').zeros(3)).cuda()
    torch.cuda.synchronize()
    print([l.split()[-1] for l in open('/proc/self/maps') if 'nvrtc' in l and 'r-xp' in l])
info(sys.argv[1])
