import sys, torch
sys.path.insert(0, ".")
import paper_1705_09864_b200 as bnn
lib = bnn.load_library()
x = torch.randn(32, 256, 28, 28, device="cuda")
out = torch.empty(32, 28, 28, 4, dtype=torch.uint64, device="cuda")
flags = torch.zeros(1, dtype=torch.int32, device="cuda")
for _ in range(5):
    lib.bnn_pack_nchw_f32(x.data_ptr(), 32, 256, 28, 28, out.data_ptr(), 0, flags.data_ptr(),
                          torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
s, e = torch.cuda.Event(True), torch.cuda.Event(True)
s.record()
for _ in range(200):
    lib.bnn_pack_nchw_f32(x.data_ptr(), 32, 256, 28, 28, out.data_ptr(), 0, flags.data_ptr(),
                          torch.cuda.current_stream().cuda_stream)
e.record(); e.synchronize()
print("eager back-to-back per launch us:", s.elapsed_time(e) / 200 * 1e3)
