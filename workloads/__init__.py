"""Seeded synthetic workloads (input spec only; none of the method's arithmetic)."""
