import numpy as np, torch, sys
sys.path.insert(0, '.')
import paper_2305_03448_b200 as desc
desc.load()
for (rows, cols, ldo, es) in [(1,1,4,4),(5,3,8,4),(3,5,4,4),(6,2,8,4),(1,1,2,8),(3,3,4,8),(33,40,36,4)]:
    dt = {4: torch.int32, 8: torch.int64}[es]
    x = torch.arange(rows*cols, dtype=dt, device='cuda').view(rows, cols) + 1
    ldi = cols + (-cols) % (16 // es)
    xin = torch.zeros((rows, ldi), dtype=dt, device='cuda'); xin[:, :cols] = x
    for k in ('tma', 'tma_st'):
        out = torch.full(((cols) * ldo + 64,), -7, dtype=dt, device='cuda')
        desc.desc_transpose_ex(xin.data_ptr(), out.data_ptr(), 1, rows, cols, ldi, ldo, 0, 0, 'f32' if es == 4 else 'f64', k)
        torch.cuda.synchronize()
        o = out.cpu().numpy()
        body = o[:cols*ldo].reshape(cols, ldo)
        print(rows, cols, ldo, es, k, 'logical ok', np.array_equal(body[:, :rows], x.cpu().numpy().T),
              'pad written', int((body[:, rows:] != -7).sum()), 'tail written', int((o[cols*ldo:] != -7).sum()))
