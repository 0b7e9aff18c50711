import sys, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen, paper_2510_13668_b200 as star
pw = datagen.make_predictor_weights(0, 4096, "bf16")
W = [torch.from_numpy(x).to(torch.bfloat16).cuda() for x in (pw.W1, pw.W2, pw.W3)]
pred = star.Predictor(*W, torch.from_numpy(pw.w4).cuda(), max_rows=512)
h = torch.from_numpy(datagen.make_hidden(0, 512, 4096)).to(torch.bfloat16).cuda()
for timing in (False, True):
    pred.layer1_timing(timing)
    y, n = star.lenpred_forward(pred, h); torch.cuda.synchronize()
    s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
    try:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            y2, n2 = star.lenpred_forward(pred, h)
        g.replay(); torch.cuda.synchronize()
        print("timing", timing, "graph ok", torch.equal(y, y2), pred.layer1_ms() if timing else None)
    except Exception as e:
        print("timing", timing, "graph FAILED", e)
