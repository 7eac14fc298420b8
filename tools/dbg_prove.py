import numpy as np, torch, sys
sys.path.insert(0,'.')
from oracle import toploc_oracle as TO
from oracle.synth_cpu import synth_bits
from paper_2505_07291_b200 import api
for H, offs in [(640,[0,45,45,110,141]), (640,[0,32]), (640,[0,13]), (640,[0,45]), (640,[0,64]), (1024,[0,45])]:
    bits = synth_bits(0, offs[-1], H, 1, 0)
    eng = api.engine()
    pb = eng.prove(torch.from_numpy(bits.view(np.int16)).cuda(), offs, return_indices=True)
    torch.cuda.synchronize()
    tab, chunks = TO._chunks_of(bits, offs, 32)
    idxs, vals, proofs = TO.prove_chunks(chunks, 128)
    gi = pb.indices.cpu().numpy(); gp = pb.proofs.cpu().numpy()
    for j in range(len(tab)):
        ok_i = np.array_equal(gi[j,:len(idxs[j])], idxs[j]); ok_p = gp[j].tobytes()==proofs[j]
        if not (ok_i and ok_p):
            print(H, offs, 'chunk', j, tab[j], 'idx ok', ok_i, 'proof ok', ok_p)
            gset=set(gi[j].tolist()); oset=set(idxs[j].tolist())
            print('   gpu-only', sorted(gset-oset)[:10], 'oracle-only', sorted(oset-gset)[:10])
            print('   gpu', gi[j][:8], 'ora', idxs[j][:8])
    print(H, offs, 'done')
