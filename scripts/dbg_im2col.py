import sys, torch
sys.path.insert(0, '.')
from paper_2603_13810_b200 import tacsnn as T, synth
spec = T.LayerSpec(T=4, B=2, C_in=2, H=128, W=128, C_out=128, pad=1, K=2, mode='tac', beta=0.5, out_pool=2, engine='tcgen05')
g = torch.Generator().manual_seed(0)
S = (torch.rand((4, 2, 2, 128, 128), generator=g) < 0.03).to(torch.uint8)
w, b = synth.weights(7, 128, 2, gain=7.1)
prep = T.prepare_weights(spec, w, b)
x = T.pack(S.cuda())
out, vf, cnt = T.conv_lif(spec, prep, x, want_v_final=True)
torch.cuda.synchronize()
print('ok', cnt.sum().item())
