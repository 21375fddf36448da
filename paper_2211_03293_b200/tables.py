"""Explicit Butcher tables used as the MRI inner integrator (textbook data,
same values and evaluation as proj/src/butcher.cpp:229-362 so the doubles are
bit-identical)."""


def _t(A, b, c, order):
    return {"A": A, "b": b, "c": c, "order": order}


def lookup_table(name: str):
    """lookup_table (proj/src/butcher.cpp:434-453) for the explicit tables."""
    if name == "heun2":  # butcher.cpp:229-240
        return _t([[0, 0], [1, 0]], [0.5, 0.5], [0, 1], 2)
    if name == "kutta3":  # butcher.cpp:242-253
        return _t([[0, 0, 0], [0.5, 0, 0], [-1, 2, 0]], [1.0 / 6.0, 2.0 / 3.0, 1.0 / 6.0],
                  [0, 0.5, 1], 3)
    if name == "bogacki-shampine3":  # butcher.cpp:258-269
        return _t([[0, 0, 0], [0.5, 0, 0], [0, 0.75, 0]], [2.0 / 9.0, 1.0 / 3.0, 4.0 / 9.0],
                  [0, 0.5, 0.75], 3)
    if name == "zonneveld4":  # butcher.cpp:274-289
        return _t([[0, 0, 0, 0, 0], [0.5, 0, 0, 0, 0], [0, 0.5, 0, 0, 0], [0, 0, 1, 0, 0],
                   [5.0 / 32.0, 7.0 / 32.0, 13.0 / 32.0, -1.0 / 32.0, 0]],
                  [1.0 / 6.0, 1.0 / 3.0, 1.0 / 3.0, 1.0 / 6.0, 0], [0, 0.5, 0.5, 1, 0.75], 4)
    if name == "classic-rk4":  # butcher.cpp:291-302
        return _t([[0, 0, 0, 0], [0.5, 0, 0, 0], [0, 0.5, 0, 0], [0, 0, 1, 0]],
                  [1.0 / 6.0, 1.0 / 3.0, 1.0 / 3.0, 1.0 / 6.0], [0, 0.5, 0.5, 1], 4)
    if name == "cash-karp5":  # butcher.cpp:304-324
        return _t([[0, 0, 0, 0, 0, 0],
                   [1.0 / 5.0, 0, 0, 0, 0, 0],
                   [3.0 / 40.0, 9.0 / 40.0, 0, 0, 0, 0],
                   [3.0 / 10.0, -9.0 / 10.0, 6.0 / 5.0, 0, 0, 0],
                   [-11.0 / 54.0, 5.0 / 2.0, -70.0 / 27.0, 35.0 / 27.0, 0, 0],
                   [1631.0 / 55296.0, 175.0 / 512.0, 575.0 / 13824.0, 44275.0 / 110592.0,
                    253.0 / 4096.0, 0]],
                  [37.0 / 378.0, 0, 250.0 / 621.0, 125.0 / 594.0, 0, 512.0 / 1771.0],
                  [0, 1.0 / 5.0, 3.0 / 10.0, 3.0 / 5.0, 1, 7.0 / 8.0], 5)
    if name == "knoth-wolke3":  # butcher.cpp:347-362
        return _t([[0, 0, 0], [1.0 / 3.0, 0, 0], [-3.0 / 16.0, 15.0 / 16.0, 0]],
                  [1.0 / 6.0, 3.0 / 10.0, 8.0 / 15.0], [0, 1.0 / 3.0, 3.0 / 4.0], 3)
    raise ValueError(f"lookup_table: unknown method '{name}'")


TABLE_NAMES = ("heun2", "kutta3", "bogacki-shampine3", "zonneveld4", "classic-rk4",
               "cash-karp5", "knoth-wolke3")
