"""One device WKT load of the canonical 1.31M-face ore text (for ncu)."""
import sys

sys.path.insert(0, ".")
import oracle as O  # noqa: E402
import paper_1808_09571_b200 as T  # noqa: E402

T.init(0)
text = O.ref_serialize_mesh(T.ore_body(1_000_000), as_bytes=True)
T.mesh_from_wkt(text)
