"""The hot path's next consumers on the device against
the reference's own implementations (oracle/_ref, built from
/root/reference/proj/src/{entropy,applications}.cpp) and the reference tests'
hand-checked cases (tests/test_entropy.cpp:60-72,
tests/test_applications.cpp:20-120)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ref():
    from oracle.oracle import Reference
    return Reference()


def test_rho_k_known_answers(knn):
    line = np.array([[0], [1], [3]], np.float32)
    assert knn.rho_k_all(line, 1).tolist() == [1.0, 1.0, 2.0]
    assert knn.rho_k_all(line, 2).tolist() == [3.0, 2.0, 3.0]
    dup = np.array([[5], [5], [9]], np.float32)
    r = knn.rho_k_all(dup, 1)
    assert r[0] == 0.0 and r[1] == 0.0 and r[2] == 4.0
    with pytest.raises(ValueError, match=r"^rho_k_all: k = 3 needs at least k \+ 1 points, set has 3$"):
        knn.rho_k_all(line, 3)


@pytest.mark.parametrize("n,d,k", [(100, 3, 4), (3000, 16, 5), (20000, 64, 20)])
def test_rho_k_all_vs_reference(knn, ref, oracle, n, d, k):
    P = oracle.uniform_f32(n, d, 1000 + d)
    got = knn.rho_k_all(P, k)
    want = ref.rho_k_all(P.astype(np.float64), k)
    assert np.allclose(got, want, rtol=1e-5, atol=0)


def test_rho_k_all_with_many_duplicates(knn, ref, oracle):
    """More than k + 1 coincident points crowd the self match out of the
    (k+1)-list: the k-th remaining entry is still 0 (entropy.cpp:48-57)."""
    base = oracle.uniform_f32(50, 8, 3)
    P = np.repeat(base, 12, axis=0)
    got = knn.rho_k_all(P, 5)
    want = ref.rho_k_all(P.astype(np.float64), 5)
    assert (got == want).all() and (got == 0).all()


def test_rho_k_all_device_pointers(knn, oracle):
    import torch
    P = oracle.uniform_f32(5000, 32, 9)
    dP = torch.from_numpy(P).cuda()
    out = torch.empty(5000, dtype=torch.float64, device="cuda")
    s = torch.cuda.Stream()
    knn.rho_k_all_device(dP.data_ptr(), 5000, 32, 7, out.data_ptr(), stream=s.cuda_stream)
    s.synchronize()
    assert (out.cpu().numpy() == knn.rho_k_all(P, 7)).all()


def test_classify_hand_checked(knn):
    assert knn.knn_classify([[0, 0], [10, 10]], [100, 200], [[1, 1]], 1).tolist() == [100]
    assert knn.knn_classify([[0, 0], [0, 1], [0, 9]], [7, 7, 8], [[0, 0.4]], 3).tolist() == [7]
    # vote tie: the smaller summed distance wins
    assert knn.knn_classify([[1], [2]], [5, 6], [[0]], 2).tolist() == [5]
    # votes and sums tie: the smaller label token wins
    assert knn.knn_classify([[-1], [1]], [9, 4], [[0]], 2).tolist() == [4]


def test_classify_contract_errors(knn):
    T = [[0, 0], [1, 1]]
    with pytest.raises(ValueError, match="exceeds reference count 2"):
        knn.knn_classify(T, [1, 2], [[0, 0]], 3)
    with pytest.raises(ValueError, match="dimension mismatch"):
        knn.knn_classify(T, [1, 2], [[0, 0, 0]], 1)
    with pytest.raises(ValueError, match="^LabeledSet: 1 labels for 2 points$"):
        knn.knn_classify([[0], [1]], [3], [[0]], 1)


@pytest.mark.parametrize("k,classes", [(1, 5), (7, 3), (20, 10), (64, 4)])
def test_classify_vs_reference(knn, ref, oracle, k, classes):
    rng = np.random.default_rng(k)
    T = oracle.uniform_f32(6000, 24, 40 + k)
    labels = rng.integers(0, classes, 6000).astype(np.int64) * 11 - 7
    Q = oracle.uniform_f32(700, 24, 50 + k)
    got = knn.knn_classify(T, labels, Q, k)
    want = ref.knn_classify(T.astype(np.float64), labels, Q.astype(np.float64), k)
    assert (got == want).all()


def test_retrieve_vote_hand_checked(knn):
    t = knn.retrieve_vote([[0, 0], [5, 5]], [0, 1], 2, [[0.1, 0]], 1)
    assert t.scores.tolist() == [1, 0] and t.ranking.tolist() == [0, 1]


def test_retrieve_vote_saturates_at_k_equal_m(knn, oracle):
    D = oracle.uniform_f32(12, 4, 1)
    own = np.repeat(np.arange(3), 4)
    Q = oracle.uniform_f32(5, 4, 2)
    t = knn.retrieve_vote(D, own, 3, Q, 12)
    assert t.scores.tolist() == [20, 20, 20] and t.ranking.tolist() == [0, 1, 2]


def test_retrieve_vote_database_errors(knn):
    D = [[0.0], [1.0]]
    with pytest.raises(ValueError, match=r"^DescriptorDatabase: image count must be >= 1$"):
        knn.retrieve_vote(D, [0, 0], 0, [[0.0]], 1)
    with pytest.raises(ValueError, match=r"^DescriptorDatabase: image identifier 5 outside \[0, 2\)$"):
        knn.retrieve_vote(D, [0, 5], 2, [[0.0]], 1)
    with pytest.raises(ValueError, match=r"^DescriptorDatabase: image 1 owns no descriptors$"):
        knn.retrieve_vote(D, [0, 0], 2, [[0.0]], 1)


@pytest.mark.parametrize("k", [1, 10, 40])
def test_retrieve_vote_vs_reference(knn, ref, oracle, k):
    rng = np.random.default_rng(k)
    images = 37
    D = oracle.uniform_f32(8000, 32, 60 + k)
    own = np.concatenate([np.arange(images), rng.integers(0, images, 8000 - images)])
    Q = oracle.uniform_f32(900, 32, 70 + k)
    t = knn.retrieve_vote(D, own, images, Q, k)
    s, r = ref.retrieve_vote(D.astype(np.float64), own, images, Q.astype(np.float64), k)
    assert (t.scores == s).all() and (t.ranking == r).all()
    assert int(t.scores.sum()) == 900 * k
