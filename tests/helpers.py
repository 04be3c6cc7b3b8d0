"""Shared fixtures for the parity tests (test infrastructure)."""
import numpy as np

from paper_2001_08743_b200 import spaces as S


def fitted(O, space, seed=0, n_train=1000):
    """(OSpace, oracle Gbt, product GbtModel) for a model fitted on SyntheticBackend samples."""
    from paper_2001_08743_b200.cost_model import GbtModel
    osp = O.OSpace(space)
    g = O.fitted_model(osp, seed=seed, n_train=n_train)
    pm = GbtModel(g.base, g.lr, g.num_features, g.offsets, g.feature, g.left, g.right, g.threshold,
                  g.value, g.training_sse)
    return osp, g, pm


def random_idx(space, n, seed):
    g = np.random.default_rng(seed)
    return np.stack([g.integers(0, c, n) for c in space.cards], 1).astype(np.int32)


def candidate_set(O, osp, n, seed, pred=None):
    """A ranked, deduplicated candidate set (CandidateSet order) of n random configs."""
    idx = random_idx(osp.space, n, seed)
    ids = osp.ids(idx)
    p = np.zeros(len(ids)) if pred is None else pred
    rows = O.make_candidate_set(osp.D, idx, ids, p, "port")
    return idx[rows], ids[rows], p[rows]


SPACES = {
    "synthetic16": lambda: S.synthetic_space(0, 16),
    "synthetic8": lambda: S.synthetic_space(7, 8),
    "resnet_c2": lambda: S.conv_space("resnet18.c2", 64, 64, 56, 56, 3, 3),
    "resnet_dense_u16": lambda: S.resnet18_tasks()[-1],
    "alexnet_c3_u16": lambda: S.alexnet_tasks()[2],
    "vgg_c4": lambda: S.vgg16_tasks()[3],
}
