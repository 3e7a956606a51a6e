import ctypes as C, os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2308_15762_b200 import _native
lib=_native.lib
lib.wp_debug_flash_fwd.argtypes=[C.c_int]*5+[C.c_void_p]*3
lib.wp_debug_flash_bwd.argtypes=[C.c_int]*5+[C.c_void_p]*7
lib.wp_debug_bw_trace.argtypes=[C.c_void_p, C.c_int]
mbs,seq,heads,d=8,1024,16,128
h=heads*d
qkv=torch.randn(mbs*seq,3*h,device='cuda').bfloat16()
ctx=torch.empty(mbs*seq,h,device='cuda',dtype=torch.bfloat16); lse=torch.empty(mbs,heads,seq,device='cuda')
dout=torch.randn(mbs*seq,h,device='cuda').bfloat16(); delta=torch.empty(mbs,heads,seq,device='cuda')
dq=torch.empty(mbs*seq,h,device='cuda'); dqkv=torch.empty(mbs*seq,3*h,device='cuda',dtype=torch.bfloat16)
lib.wp_debug_flash_fwd(mbs,seq,heads,d,1,qkv.data_ptr(),ctx.data_ptr(),lse.data_ptr())
for _ in range(3):
    lib.wp_debug_flash_bwd(mbs,seq,heads,d,1,qkv.data_ptr(),ctx.data_ptr(),dout.data_ptr(),lse.data_ptr(),delta.data_ptr(),dq.data_ptr(),dqkv.data_ptr())
buf=(C.c_ulonglong*512)()
lib.wp_debug_bw_trace(buf,512)
N={12:'sm_wait_dP',13:'sm_got_dP',1:'mma_dP_committed',2:'mma_S_committed',3:'mma_got_dS',4:'mma_dQ_committed',5:'sm_wait_S',6:'sm_got_S',7:'sm_dS_ready',8:'dq_wait',9:'dq_got',10:'dq_drained',11:'mma_got_dqfree'}
ev=sorted((buf[e*32+j],e,j) for e in range(16) for j in range(32) if buf[e*32+j])
t0=ev[0][0]
for t,e,j in ev: print(f"{t-t0:8d} it={j:2d} {N.get(e,e)}")
