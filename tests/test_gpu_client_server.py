"""GPU: client / server split. A secret-holding context exports its
evaluation keys (lv_keys_export); an evaluation-only context built from them
(lv_ctx_create_eval) runs every homomorphic entry point without a secret
key and produces ciphertexts bit-identical to the client's own."""
import numpy as np
import pytest

import paper_2508_14568_b200 as L
from paper_2508_14568_b200 import leuven as LV

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def split():
    client = L.Context(seed=3)
    bsk, ksk, kid = client.export_keys()
    server = L.Context.evaluation(bsk, ksk, kid)
    yield client, server
    server.close()
    client.close()


def test_exported_keys_equal_oracle(ctx, orc):
    bsk, ksk, kid = ctx.export_keys()
    assert kid not in (0, 1)  # a fingerprint of public material, never the seed (0 here)
    assert np.array_equal(ksk, orc.ksk())
    assert np.array_equal(bsk, orc.bsk())


def test_server_has_no_secret(split):
    _, server = split
    with pytest.raises(L.InvalidParams):
        server.encrypt([1])
    t = server.trivial([5])
    with pytest.raises(L.InvalidParams):
        server.decrypt(t)
    with pytest.raises(L.InvalidParams):
        server.export_keys()
    with pytest.raises(L.InvalidParams):
        L.Context.evaluation(np.zeros(10, np.uint64), np.zeros(10, np.uint64), 0)


def test_key_id_is_public_fingerprint(split):
    """the key id must not be the generating seed (anyone holding
    a table file could regenerate the secret key from it). It is a hash of
    the public KSK + parameters: equal on client and server, different per
    key set, and a server rejects keys that do not match an announced id."""
    client, server = split
    bsk, ksk, kid = client.export_keys()
    assert kid != 3
    assert server.key_id() == kid
    other = L.Context(seed=4)
    assert other.export_keys()[2] != kid
    other.close()
    with pytest.raises(L.InvalidParams):
        L.Context.evaluation(bsk, ksk, kid ^ 1)


def test_server_pbs_bit_identical(split, golden):
    client, server = split
    lut = golden["luts"]["minlut-negated"]
    vals = list(range(32)) * 3
    cts = client.encrypt(vals)
    rows = client.export(cts)
    mine = client.export(client.pbs(cts, lut))
    theirs = server.export(server.pbs(server.import_(rows), lut))
    assert np.array_equal(mine, theirs)
    back = client.import_(theirs)
    assert list(client.decrypt(back)) == [L.negacyclic_eval(lut, v) for v in vals]
    # the host-buffer path on the server, too
    ids = np.full(len(vals), server.lut(lut), np.uint32)
    assert np.array_equal(server.pbs_host(rows, ids), mine)


def test_server_edit_distance(split):
    client, server = split
    spec = LV.AlphabetSpec.ascii7()
    a, b = "monday", "friday"
    xa = LV.encrypt_string(a, spec, client)
    xb = LV.encrypt_string(b, spec, client)
    # ship the symbol ciphertexts to the server, compute there, ship the score back
    sa = LV.EncryptedString(server.import_(client.export(xa.chars.reshape(-1))).reshape(xa.chars.shape))
    sb = LV.EncryptedString(server.import_(client.export(xb.chars.reshape(-1))).reshape(xb.chars.shape))
    run = LV.distance_encrypted(server, sa, sb, LV.BandSpec.exact(len(a), len(b)))
    assert (run.kernel_pbs, run.equality_pbs) == (36, 72)
    score = client.import_(server.export([run.score]))
    assert list(client.decrypt(score)) == [LV.wf_distance(a, b)]


def test_server_eq_table_travels_to_client(split, tmp_path):
    client, server = split
    spec = LV.AlphabetSpec.dna4()
    q = "ACGTTGCA"
    xq = LV.encrypt_string(q, spec, client)
    sq = LV.EncryptedString(server.import_(client.export(xq.chars.reshape(-1))).reshape(xq.chars.shape))
    table, pbs = LV.build_eq_table(server, sq, spec)
    assert pbs == len(spec.charset()) * len(q)
    path = tmp_path / "q.leqt"
    LV.save_eq_table(table, path)
    # the key-set id in the file is the client's: the client accepts it
    mine = LV.load_eq_table(client, path)
    run = LV.distance_preprocessed(client, mine, "ACGATGC", LV.BandSpec.exact(len(q), 7))
    assert list(client.decrypt([run.score])) == [LV.wf_distance(q, "ACGATGC")]
