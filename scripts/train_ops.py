"""Which torch ops run inside one training step (bench.py --train glue + TrainableNetwork)?"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from paper_2603_13810_b200 import configs, network, tacsnn  # noqa: E402

cfg = configs.CONFIGS["C4"]
B = 16
specs = configs.layer_plan(cfg, mode="tactp", K=2, B=B)
net = network.TrainableNetwork(specs, configs.layer_weights(cfg), surrogate="arctan", alpha=2.0, detach_reset=True)
x = tacsnn.pack(configs.make_inputs(cfg, B=B, device="cuda"))


def step():
    _, cnt, tape = net.forward_train(x)
    s_last = tape[-1][0]
    hc, wc = s_last.conv_hw
    T_out = tape[-1][4].shape[0]
    err = (cnt.float() / float(T_out * hc * wc)) / float(T_out * hc * wc)
    g_out = err[None, :, None, None, :].expand(T_out, B, hc, wc, s_last.C_out).contiguous()
    return net.backward(tape, g_out)


step()
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CPU, torch.profiler.ProfilerActivity.CUDA]) as prof:
    step()
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=25))
