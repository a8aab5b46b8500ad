"""pytest plugin (``-p headbalance_plugin`` with tests/dropin on sys.path): before the
reference's conftest imports ``headbalance``, make that name resolve to this
package composed with the reference's off-hot-path modules
(tests/dropin/compose.py).  TEST INFRASTRUCTURE ONLY."""

from compose import alias_as_headbalance

alias_as_headbalance()
