"""Timeline of CTA 0 of the attention backward (library built with
-DWP_BW_TRACE, e.g. a `#define WP_BW_TRACE 1` atop attention_bwd.cu): per
(event, q tile) SM clock in time order.  CAUSAL=1 for the causal kernel."""
import ctypes as C, os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2308_15762_b200 import _native
lib=_native.lib
lib.wp_debug_flash_fwd.argtypes=[C.c_int]*5+[C.c_void_p]*3
lib.wp_debug_flash_bwd.argtypes=[C.c_int]*5+[C.c_void_p]*7
lib.wp_debug_bw_trace.argtypes=[C.c_void_p, C.c_int]
mbs,seq,heads,d=16,1024,16,int(os.environ.get('D','128'))
causal=int(os.environ.get('CAUSAL','0'))
h=heads*d
qkv=torch.randn(mbs*seq,3*h,device='cuda').bfloat16()
ctx=torch.empty(mbs*seq,h,device='cuda',dtype=torch.bfloat16); lse=torch.empty(mbs,heads,seq,device='cuda')
dout=torch.randn(mbs*seq,h,device='cuda').bfloat16(); delta=torch.empty(mbs,heads,seq,device='cuda')
dq=torch.empty(mbs*seq,h,device='cuda'); dqkv=torch.empty(mbs*seq,3*h,device='cuda',dtype=torch.bfloat16)
lib.wp_debug_flash_fwd(mbs,seq,heads,d,causal,qkv.data_ptr(),ctx.data_ptr(),lse.data_ptr())
for _ in range(3):
    lib.wp_debug_flash_bwd(mbs,seq,heads,d,causal,qkv.data_ptr(),ctx.data_ptr(),dout.data_ptr(),lse.data_ptr(),delta.data_ptr(),dq.data_ptr(),dqkv.data_ptr())
buf=(C.c_ulonglong*832)()
lib.wp_debug_bw_trace(buf,832)
N={13:'dq_got_h1',14:'mma_dQh0_issued',15:'mma_dQh1_issued',1:'mma_got_dS',2:'mma_dQ_committed',3:'mma_S_issued',12:'mma_dV_issue(p_full)',4:'mma_dP_issue(dqfree,dO)',5:'sm_got_S',6:'sm_phaseA_done',7:'sm_got_dP',8:'sm_got_pdsfree',9:'sm_dS_arrived',10:'dq_got',11:'dq_free_arrive'}
ev=sorted((buf[e*32+j],e,j) for e in range(16) for j in range(32) if buf[e*32+j])
t0=ev[0][0]
for t,e,j in ev: print(f"{t-t0:8d} it={j:2d} {N.get(e,e)}")
cta=[(buf[512+2*i],buf[513+2*i]) for i in range(148) if buf[512+2*i]]
if cta:
    t0=min(a for a,b in cta); durs=sorted(b-a for a,b in cta); ends=sorted(b-t0 for a,b in cta)
    print(f"CTAs {len(cta)}: duration min {durs[0]/1e3:.1f} us  median {durs[len(durs)//2]/1e3:.1f}  max {durs[-1]/1e3:.1f}; "
          f"end spread {ends[0]/1e3:.1f}..{ends[-1]/1e3:.1f} us; starts spread {(max(a for a,b in cta)-t0)/1e3:.1f} us")
