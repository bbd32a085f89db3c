"""Placement communication ledgers: dgnn_comm_ledger against
the CommLedger of the reference's own run_distributed_epoch
(src/distsim.cpp:101-182, 262-268) for every placement scheme and overlap
mode — byte counts must be identical."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

# stride 3 keeps the last window's target inside [0, T) so the reference's
# distributed epoch can run (it windows the full length)
GRAPH = dict(n=300, avg_degree=4, dim=8, T=12, edge=0.05, feat=0.02)


@pytest.fixture(scope="module")
def pair(ref):
    import torch
    assert torch.cuda.is_available()
    from paper_2501_15348_b200 import api
    g = GRAPH
    args = (g["n"], g["avg_degree"], g["dim"], g["T"], g["edge"], g["feat"])
    return api, ref.RefGraph.synth(*args, seed=2), api.Synth(*args, seed=2).to_graph()


SCHEMES = ["consecutive_block", "node_partition", "sequence_partition"]
OVERLAPS = ["replicate_overlap", "remote_fetch"]


@pytest.mark.parametrize("scheme", range(3))
@pytest.mark.parametrize("overlap", range(2))
@pytest.mark.parametrize("workers,batch", [(1, 0), (2, 0), (3, 100)])
def test_ledger_matches_reference(pair, ref, scheme, overlap, workers, batch):
    api, gr, g = pair
    cfg = ref.RunCfg(arch="gcrn_m2", hidden=16, seq_len=3, stride=3, workers=workers,
                     batch_size=batch, optimizer="sgd")
    want, npar, nb = gr.comm_ledger(cfg, scheme, overlap)
    got = api.comm_ledger(g, SCHEMES[scheme], OVERLAPS[overlap], workers=workers, seq_len=3,
                          stride=3, horizon=1, hidden=16, num_params=npar, num_batches=nb)
    assert np.array_equal(got, want), (got, want)
    if workers > 1:  # one worker communicates nothing
        assert got[-1].sum() > 0
