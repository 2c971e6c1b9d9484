"""Seeded synthetic input generators shared by tests and bench (no method arithmetic)."""
