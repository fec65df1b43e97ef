"""Version of the B200 engine behind the ``sparseconv`` mirror."""

from paper_2204_10319_b200 import __version__  # noqa: F401
