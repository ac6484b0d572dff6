"""fp32 stem conv (7x7/2, 3->64, 224^2, batch 256): cuDNN NCHW vs channels_last, TF32 off."""
import torch
torch.backends.cudnn.allow_tf32 = False
torch.backends.cuda.matmul.allow_tf32 = False
torch.backends.cudnn.benchmark = True
x = torch.randn(256, 3, 224, 224, device="cuda")
w = torch.randn(64, 3, 7, 7, device="cuda")
def t(fn, n=5):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(n): fn()
    e.record(); e.synchronize()
    return s.elapsed_time(e) / n
f = torch.nn.functional.conv2d
print("nchw ms", t(lambda: f(x, w, stride=2, padding=3)))
xc, wc = x.to(memory_format=torch.channels_last), w.to(memory_format=torch.channels_last)
print("nhwc ms", t(lambda: f(xc, wc, stride=2, padding=3)))
y1 = f(x, w, stride=2, padding=3); y2 = f(xc, wc, stride=2, padding=3)
print("max |diff| nchw vs nhwc", (y1 - y2).abs().max().item())
# reference: fp64 on a slice
y64 = f(x[:2].double(), w.double(), stride=2, padding=3)
print("max rel err nchw", ((y1[:2].double() - y64).abs().max() / y64.abs().max()).item(), "nhwc", ((y2[:2].double() - y64).abs().max() / y64.abs().max()).item())
