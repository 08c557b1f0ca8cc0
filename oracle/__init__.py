"""CPU oracle of the reference OptV2 path — TEST INFRASTRUCTURE ONLY.

Importable only from tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs.
The product package paper_1305_3122_b200 must never import it.
"""
