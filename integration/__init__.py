"""Reference-side bindings of the B200 C ABI."""
