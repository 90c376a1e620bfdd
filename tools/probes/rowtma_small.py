import sys, torch
sys.path.insert(0, ".")
import paper_2601_11608_b200 as wf
for (n,h,w,k,co,s,p) in [(2,40,53,5,96,1,0),(3,227,227,11,96,4,0)]:
    torch.manual_seed(0)
    x = torch.randint(-4,5,(n,h,w,3),device="cuda").bfloat16()
    wt = torch.randint(-4,5,(k,k,3,co),device="cuda").bfloat16()
    conv = wf.FoldedConv2d(wt, None, x.shape, stride=s, padding=p)
    print(conv.device_plan["producer"], conv.device_plan["n_tiles"], flush=True)
    y = conv(x, out_dtype=torch.float32); torch.cuda.synchronize()
    ref = torch.nn.functional.conv2d(x.double().permute(0,3,1,2), wt.double().permute(3,2,0,1), stride=s, padding=p).permute(0,2,3,1)
    print("exact:", torch.equal(y.double(), ref), flush=True)
