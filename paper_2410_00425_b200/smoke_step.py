"""Placeholder hook for the step/render smoke check (grows with the engine)."""


def run() -> None:
    return None
