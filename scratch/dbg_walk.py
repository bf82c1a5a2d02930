def terms(f, i):
    return list(zip(f.feat[f.term_off[i]:f.term_off[i+1]].tolist(), f.weight[f.term_off[i]:f.term_off[i+1]].tolist()))
def size(f, i):
    return 1 if f.left[i] < 0 else 1 + size(f, f.left[i]) + size(f, f.right[i])
def walk(a, b, i, j, depth, path):
    if (a.left[i] < 0) != (b.left[j] < 0) or a.thr[i].tobytes() != b.thr[j].tobytes() or terms(a, i) != terms(b, j) or a.pred[i] != b.pred[j]:
        return (depth, path, "gpu", int(a.left[i]), repr(a.thr[i]), terms(a, i)[:4], int(a.pred[i]), "ref", int(b.left[j]), repr(b.thr[j]), terms(b, j)[:4], int(b.pred[j]), "subtree", size(b, j))
    if a.left[i] < 0: return None
    return walk(a, b, a.left[i], b.left[j], depth + 1, path + "L") or walk(a, b, a.right[i], b.right[j], depth + 1, path + "R")
