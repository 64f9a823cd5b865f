"""Host-side containers mirror chunk.hpp / collection.hpp (restating test_chunk.cpp and
test_collection.cpp expectations)."""
import numpy as np

from conftest import golden


def test_chunk_layout_worked_example(ssj):
    # test_chunk.cpp:9-35 (paper Fig 5)
    b = ssj.ChunkBuilder()
    b.append(1, [9])
    b.append(2, [])
    b.append(3, [4, 7])
    chunk = b.seal()
    assert chunk.C.tolist() == [9, 4, 7]
    assert chunk.C_O.tolist() == [1, 1, 2, 1, 3, 3]
    assert chunk.candidate_count() == 3
    assert chunk.byte_size() == 36
    sl = ssj.decode(chunk)
    assert [s.probe for s in sl] == [1, 2, 3]
    assert sl[0].begin == 0 and sl[0].candidates.tolist() == [9]
    assert sl[1].candidates.size == 0
    assert sl[2].begin == 1 and sl[2].candidates.tolist() == [4, 7]


def test_builder_capacity_accounting(ssj):
    # test_chunk.cpp:37-52
    B = ssj.ChunkBuilder
    b = B(B.kEntryBytes + 2 * B.kCandidateBytes)
    assert b.capacity() == 2 and b.entry_fits()
    b.append(0, [5, 6])
    assert b.capacity() == 0 and not b.entry_fits()
    assert b.byte_size() == b.budget()
    chunk = b.seal()
    assert chunk.candidate_count() == 2 and b.empty() and b.capacity() == 2


def test_zero_width_entries(ssj):
    # test_chunk.cpp:54-64
    B = ssj.ChunkBuilder
    b = B(2 * B.kEntryBytes)
    b.append(0, [])
    assert b.entry_fits() and b.capacity() == 0
    b.append(1, [])
    assert not b.entry_fits()
    chunk = b.seal()
    assert chunk.C.size == 0 and len(ssj.decode(chunk)) == 2


def test_chunk_round_trip_property(ssj):
    # test_chunk.cpp:66-98
    rng = np.random.default_rng(3)
    for _ in range(200):
        budget = ssj.ChunkBuilder.kMinBudget + int(rng.integers(0, 4096))
        b = ssj.ChunkBuilder(budget)
        written = []
        probe = 0
        while b.entry_fits():
            cap = b.capacity()
            take = int(rng.integers(0, cap + 1)) if cap else 0
            cands = rng.integers(0, 1000, size=take).astype(np.uint32)
            b.append(probe, cands)
            written.append((probe, cands))
            probe += 1
        assert b.byte_size() <= budget
        chunk = b.seal()
        assert chunk.byte_size() <= budget
        sl = ssj.decode(chunk)
        cursor = 0
        for s, (p, c) in zip(sl, written):
            assert s.probe == p and s.begin == cursor and np.array_equal(s.candidates, c)
            cursor += c.size
        assert cursor == chunk.candidate_count()


def test_preprocess_precoded_order(ssj):
    # collection.hpp:134-168: dedup, sort, drop empties, order by (size, lex, line)
    recs = [[5, 3, 3], [], [1], [2, 9], [3, 5], [7]]
    c = ssj.preprocess_precoded(recs)
    assert c.dropped_empty == 1
    sets = [c.set_view(i).tolist() for i in range(c.size())]
    assert sets == [[1], [7], [2, 9], [3, 5], [3, 5]]
    assert c.original_id.tolist() == [2, 5, 3, 0, 4]
    assert c.average_set_size() == 8 // 5


def test_collection_matches_reference_layout(ssj):
    g = golden("verify_s41")
    c = ssj.Collection(g["tokens"], g["offsets"], g["original_id"])
    assert c.size() == 200
    for i in range(c.size()):
        v = c.set_view(i)
        assert np.all(np.diff(v.astype(np.int64)) > 0)
    sizes = np.diff(c.offsets.astype(np.int64))
    assert np.all(np.diff(sizes) >= 0)
