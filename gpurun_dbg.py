import numpy as np, torch, eg_inputs as G, oracle as O, paper_2303_02724_b200 as eg
ctx = eg.Context()
for dims, kind in [([70, 9, 40], "signed_zero"), ([33, 35, 19], "int"), ([65, 33, 17], "normal")]:
    f, _ = G.random_field(dims, 17 + len(dims), kind)
    o = O.grid(f, dims)
    t = torch.from_numpy(f).cuda()
    bad = 0
    for it in range(30):
        g = ctx.compute(t, dims=dims)
        lab = g.labels.cpu().numpy()
        d = np.nonzero(lab != o.label)[0]
        st = ctx.stats()
        if len(d):
            bad += 1
            if bad < 4:
                v = d[0]
                print(dims, kind, "iter", it, "ndiff", len(d), "v", v, "gpu", lab[v], "oracle", o.label[v], "ptr_oracle", o.ptr[v], "exit_targets", st["n_exit_targets"])
    print(dims, kind, "bad runs", bad, "/30")
