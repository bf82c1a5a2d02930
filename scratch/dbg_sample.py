import sys, numpy as np
sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import oracle_lib, paper_2603_00326_b200 as sofg
o = oracle_lib.get('reference')
ctx = sofg.Context(0)
for d in (64, 512, 4096):
    R,_,dens = o.projection_config(d)
    seeds = np.array([o.derive_seed(7,i) for i in range(300)], np.uint64)
    skips = np.array([(i*13)%700 for i in range(300)], np.uint64)
    rp,feat,w,used = ctx.sample_projection(d,R,dens,seeds,skips)
    bad=[]
    for i in range(300):
        orp,ofeat,ow,oused = o.sample_projection(d,R,dens,int(seeds[i]),int(skips[i]))
        z=int(orp[-1])
        ok = np.array_equal(rp[i],orp) and np.array_equal(feat[i,:z],ofeat) and int(used[i])==oused
        if not ok:
            zb, ub = o.binomial_draw(R*d, dens, int(seeds[i]), int(skips[i]))
            # python Floyd draws
            outs = o.rng_outputs(int(seeds[i]), ub, z)
            cells=R*d
            t=[(int(outs[q])*(cells-z+q+1))>>64 for q in range(z)]
            bad.append((i,int(skips[i]),ub,z,len(set(t))<z, int(used[i]), oused))
    print(d, len(bad), bad[:12])
